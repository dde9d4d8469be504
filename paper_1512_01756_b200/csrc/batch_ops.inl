// Operators on device vectors (part of batch.cu's translation unit).
// Included by batch.cu; not a standalone header.
// --------------------------------------------------------------------------
// Operators (device vectors nsys x k)
// --------------------------------------------------------------------------
void op_S(smpm_batch* b, const double* v, double* y, const Live& lv, cudaStream_t st) {
  ProfScope ps(b, PC_SCHUR, st);
  run_plan(b, b->pS, v, y, nullptr, lv, st);
}
void op_St(smpm_batch* b, const double* v, double* y, const Live& lv, cudaStream_t st) {
  run_plan(b, b->pSt, v, y, nullptr, lv, st);
}
// structured block-Jacobi: three dependent GEMM stages
void op_BJ(smpm_batch* b, const double* v, double* y, const Live& lv, cudaStream_t st) {
  ProfScope ps(b, PC_BJ, st);
  double* tmp = b->vbuf[9].p;
  run_plan(b, b->pBJ1, v, y, tmp, lv, st);
  run_plan(b, b->pBJ2, v, y, tmp, lv, st);
  run_plan(b, b->pBJ3, v, y, tmp, lv, st);
}
// P v = v - S Z c(Z^T v)
void op_P(smpm_batch* b, const double* v, double* y, bool fused, const Live& lv, cudaStream_t st) {
  if (fused) {
    run_deflate(b, DEFL_P_FUSED, v, v, y, nullptr, lv, st);
    return;
  }
  double* c = b->dsmall.p;
  double* z = b->vbuf[7].p;
  double* sz = b->vbuf[8].p;
  run_deflate(b, DEFL_COARSE, v, nullptr, nullptr, c, lv, st);
  zbroadcast_kernel<<<grid_for(b->nsys * b->k), 256, 0, st>>>(b->nsys, b->d, 2 * b->w, b->k, lv.active, c, z);
  check_launch(b);
  op_S(b, z, sz, lv, st);
  run_deflate(b, DEFL_SUB_T, sz, v, y, nullptr, lv, st);
}
// Q v = v - Z c(Z^T S v)
void op_Q(smpm_batch* b, const double* v, double* y, const Live& lv, cudaStream_t st) {
  double* t = b->vbuf[8].p;
  op_S(b, v, t, lv, st);
  run_deflate(b, DEFL_Q_TAIL, t, v, y, nullptr, lv, st);
}
