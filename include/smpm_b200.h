/*
 * smpm_b200.h — C ABI of the B200-native deflated block-Jacobi Schur-GMRES
 * solve (SMPM Poisson-Neumann / per-Fourier-mode Helmholtz).
 *
 * Drop-in boundary for the reference library `smpm` (C++20/Eigen,
 * /root/reference/proj). Each entry point replaces the reference routine
 * cited beside it. Plain pointers and sizes only; no torch types.
 *
 * Layout conventions:
 *  - A *batch* holds `nsys` independent Schur systems of one geometry
 *    (n GLL points, m_x strips, m_z elements per strip): the 2D Poisson
 *    system (nsys = 1) or the per-wavenumber systems of the Fourier
 *    extension. w = n*m_z, d = m_x-1 interfaces, k = 2*w*d interface slots.
 *  - Interface vectors use the reference slot order
 *    (/root/reference/proj/include/smpm/mesh.hpp:43-47): slot
 *    i*2w + side*w + ez*n + iz. Batched vectors are nsys x k, system-major,
 *    contiguous. Coarse vectors are nsys x d.
 *  - Coupling matrices are column-major (Eigen default) per strip kind:
 *    G_W (w x w)   west-boundary strip: east-readers x east-own columns
 *    G_I (2w x 2w) interior strip: rows [west-readers; east-readers],
 *                  cols [west-own; east-own]
 *    G_E (w x w)   east-boundary strip: west-readers x west-own columns
 *    exactly the per-kind block `build_kind_coupling` produces
 *    (/root/reference/proj/src/schur.cpp:19-69).
 *  - Vector arguments of the operator entry points are DEVICE pointers
 *    (cudaMalloc'd, 16-byte aligned); `stream` is a cudaStream_t (NULL =
 *    the context's stream). The *_host solve entry points take host
 *    pointers and include the copies.
 *
 * Errors: every call returns an smpm_status; smpm_last_error() describes the
 * last failure on the calling thread. SMPM_EINVAL mirrors the reference's
 * std::invalid_argument, SMPM_ENONFINITE / SMPM_ESINGULAR / SMPM_ERUNTIME
 * its std::runtime_error cases; non-convergence is reported in
 * smpm_report.converged, never as an error (proj/src/gmres.cpp:137).
 * There is no CPU fallback: without a usable sm_100 device every call that
 * needs one fails with SMPM_ECUDA.
 */
#ifndef SMPM_B200_H
#define SMPM_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SMPM_OK = 0,
  SMPM_EINVAL = 1,
  SMPM_ERUNTIME = 2,
  SMPM_ENONFINITE = 3,
  SMPM_ESINGULAR = 4,
  SMPM_ECUDA = 5,
  SMPM_ENCCL = 6
} smpm_status;

/* proj/include/smpm/solver.hpp:11 (Method) */
typedef enum { SMPM_SCHUR = 0, SMPM_BJ = 1, SMPM_DBJ = 2, SMPM_2LAS = 3 } smpm_method;

/* Arnoldi orthogonalization used on the device. The reference uses
 * Householder reflections (proj/src/gmres.cpp:58-68); both variants span the
 * same Krylov space. */
typedef enum { SMPM_ORTH_CGS2 = 0, SMPM_ORTH_MGS = 1 } smpm_orth;

typedef struct smpm_ctx smpm_ctx;
typedef struct smpm_batch smpm_batch;

/* proj/include/smpm/gmres.hpp:20-28 (KrylovReport) + proj/include/smpm/deflation.hpp:44-48 */
typedef struct {
  int iterations;
  int converged;
  int mismatch_warning;
  int history_len;                /* entries written to the history buffer */
  long long operator_applies;
  long long krylov_s_applies;     /* S applications inside the GMRES call */
  double final_rel_residual;
  double wall_time_s;             /* device time of the whole batched solve */
} smpm_report;

/* proj/include/smpm/gmres.hpp:12-18 (GmresOptions) + driver arguments of
 * deflated_solve / two_level_schwarz_solve (proj/include/smpm/deflation.hpp:55-61) */
typedef struct {
  double tol;          /* relative to ||b_S|| (proj/src/deflation.cpp:109) */
  int max_iter;        /* total Arnoldi steps */
  int restart;         /* 0 = never restart (reference); m = GMRES(m) */
  int orth;            /* smpm_orth */
  int fuse_deflation;  /* 1: P applied through O(k) row-sum identities (one S per dbj step); 0: literal */
  int final_residual_check; /* 1 as the reference default */
} smpm_solve_options;

const char* smpm_last_error(void);
/* version string incl. the arch the kernels were built for */
const char* smpm_version(void);

/* ---- context / batch lifecycle ------------------------------------------ */
int smpm_ctx_create(int device, smpm_ctx** out);
int smpm_ctx_destroy(smpm_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) */
void* smpm_ctx_stream(smpm_ctx* ctx);

int smpm_batch_create(smpm_ctx* ctx, int n, int m_x, int m_z, int nsys, smpm_batch** out);
int smpm_batch_destroy(smpm_batch* b);
/* k, d, w of the batch geometry */
int smpm_batch_dims(const smpm_batch* b, long long* k, int* d, int* w);

/* Per-kind couplings of system `sys` (host pointers, column-major, see
 * layout above). Replaces the interface-block storage of SchurSystem
 * (proj/include/smpm/schur.hpp:32-36): the reference copies these blocks
 * verbatim into every interface (proj/src/schur.cpp:113-124). G_I is
 * ignored when m_x == 2. */
int smpm_batch_set_couplings(smpm_batch* b, int sys, const double* G_W, const double* G_I, const double* G_E);

/* Reference-layout import: the d interface blocks of one SchurSystem
 * (proj/include/smpm/schur.hpp:32-36 / dump format proj/src/schur.cpp:246-297):
 * entries[i] is column-major rows_i x 2w, segment starts/lengths as in
 * InterfaceBlock::row_segments. The blocks are verified to be copies of at
 * most three strip-kind couplings and deduplicated into them. */
int smpm_batch_set_interface_blocks(smpm_batch* b, int sys, const double* const* entries, const long long* rows,
                                    const long long* const* seg_start, const long long* const* seg_len,
                                    const int* nseg);

/* Reads the reference's binary block file (dump_schur_blocks, proj/src/schur.cpp:246-297:
 * int64 n, m_x, m_z, k; per interface block rows, cols, nseg, (start, len) x nseg,
 * column-major entries) for system `sys` and imports it as set_interface_blocks does. */
int smpm_batch_load_schur_blocks(smpm_batch* b, int sys, const char* path);

/* Left null vector u_S of a singular system (the j = 0 / Poisson system):
 * marks the system singular; the coarse solve uses the rank-one shift
 * (C + u_C u_C^T) with u_C = normalize(Z^T u_S) (proj/src/deflation.cpp:44-54). */
int smpm_batch_set_nullspace(smpm_batch* b, int sys, const double* u_S);

/* Optional spectral factors of the couplings (before finalize).  Every
 * coupling block is G_kind[X,Y] = T diag_q(gamma_kind,XY) T^{-1} in the real
 * eigenbasis T (w x w, column-major) of the strip operator's z factor, with
 * the `npairs` complex-conjugate eigenpairs first (columns Re v, Im v) and the
 * w - 2 npairs real modes after; a pair's gamma acts on z = a - i b.  gamma is
 * nsys x 6 x nmode complex numbers (re, im interleaved; nmode = w - npairs) in
 * kind order W_EE, I_WW, I_WE, I_EW, I_EE, E_WW (G_W = W_EE; G_I = [[I_WW,
 * I_WE], [I_EW, I_EE]]; G_E = E_WW).  The dense couplings stay the reference
 * data (set_couplings is still required); with factors set, the Krylov
 * operator runs as two shared-matrix GEMMs (T^{-1}, T) around per-mode work
 * (the fast-diagonalisation form of the A^{-1}B sweep), with identical
 * results up to rounding.  Replaces nothing in the reference API; it is the
 * data the reference computes in build_kind_coupling (proj/src/schur.cpp:19-69)
 * before densifying it. */
int smpm_batch_set_spectral(smpm_batch* b, int npairs, const double* T, const double* T_inv, const double* gamma);

/* Uploads, builds the block-Jacobi inverses (proj/src/schur.cpp:188-216),
 * the coarse matrices C = Z^T S Z and their solvers (proj/src/deflation.cpp:24-69). */
int smpm_batch_finalize(smpm_batch* b);

/* Coarse matrices (nsys x d x d, column-major) and tridiagonal flags, host out */
int smpm_batch_coarse_info(smpm_batch* b, double* C, int* tridiagonal, int* singular);

/* ---- operators: device pointers, nsys x k (x_d: nsys x d) ----------------- */
int smpm_apply_S(smpm_batch* b, const double* v, double* y, void* stream);                 /* proj/src/schur.cpp:143-158 */
int smpm_apply_St(smpm_batch* b, const double* v, double* y, void* stream);                /* proj/src/schur.cpp:160-175 */
int smpm_apply_block_jacobi_inv(smpm_batch* b, const double* v, double* y, void* stream);  /* proj/src/schur.cpp:218-225 */
int smpm_apply_Z(smpm_batch* b, const double* y_d, double* v, void* stream);               /* proj/src/deflation.cpp:8-14 */
int smpm_apply_Zt(smpm_batch* b, const double* v, double* y_d, void* stream);              /* proj/src/deflation.cpp:16-22 */
int smpm_coarse_solve(smpm_batch* b, const double* b_d, double* x_d, void* stream);        /* proj/src/deflation.cpp:71-92 */
int smpm_apply_P(smpm_batch* b, const double* v, double* y, int fused, void* stream);      /* proj/src/deflation.cpp:94-96 */
int smpm_apply_Q(smpm_batch* b, const double* v, double* y, void* stream);                 /* proj/src/deflation.cpp:98-100 */
/* out = v - dir (dir . v) per system; v, dir, out are nsys x len, any len >= 1:
 * u_S on b_S (len = k) or u_L on f (len = r) (proj/src/nullspace.cpp:92). */
int smpm_project_out(smpm_batch* b, long long len, const double* v, const double* dir, double* out, void* stream);

/* ---- strip solves either side of the path --------------
 * Fast-diagonalisation factors of the strip operator A - mu I.  The reference
 * LU-factors every strip kind (proj/src/operator.cpp:113-124) and real-Schur
 * factors the Helmholtz shifts (proj/src/helmholtz.cpp:58-87); every strip
 * block is the Kronecker sum Ax_kind (x) I + I (x) Az with Az shared by all
 * kinds and diagonalised by the spectral basis T of smpm_batch_set_spectral,
 * so a strip solve is, per z mode, an n x n complex solve along x.  Complex
 * numbers are (re, im) interleaved; matrices column-major. */
typedef struct {
  const double* Vx[3];     /* per strip kind (0: west-boundary strip, 1: interior, 2: east-boundary):
                              eigenvectors of Ax_kind, n x n complex */
  const double* Vx_inv[3]; /* their inverses, n x n complex */
  const double* lx[3];     /* eigenvalues of Ax_kind, n complex */
  const double* lz;        /* eigenvalues of Az in the spectral basis order (per complex pair the member
                              with Im > 0, then the real modes): w - npairs complex */
  const double* tW;        /* n: west-edge trace weights of B = -tau t_X . u (proj/src/operator.cpp:127-151) */
  const double* tE;        /* n: east-edge trace weights */
  double tau;              /* penalty (proj/src/operator.cpp:78-82) */
  const double* mu;        /* nsys Helmholtz shifts k_j^2 (0: Poisson) */
} smpm_strip_factors;
int smpm_batch_set_strip_factors(smpm_batch* b, const smpm_strip_factors* f);
/* Device-side per-mode setup: INSTEAD of per-system couplings
 * (smpm_batch_set_couplings) and spectral diagonals (smpm_batch_set_spectral) the
 * caller hands over the geometry-level fast-diagonalisation factors once — the
 * shared z eigenbasis T, T^{-1} (w x w, column-major, npairs complex pairs first)
 * and the strip factors with the per-system shifts mu — and smpm_batch_finalize
 * builds, with this library's own kernels, for every system: the spectral
 * diagonals gamma(mu), the dense couplings G_kind = T diag(gamma) T^{-1}
 * (replacing build_kind_coupling's LU per kind, proj/src/schur.cpp:19-69, and the
 * per-shift real-Schur solves, proj/src/helmholtz.cpp:58-143), the block-Jacobi
 * inverses K^{-1} = T diag(kinv) T^{-1} (replacing the LU of build_block_jacobi,
 * proj/src/schur.cpp:188-216), the strip row sums and the coarse matrix
 * (proj/src/deflation.cpp:24-69).  Also stores the strip factors (as
 * smpm_batch_set_strip_factors).  Needs w % 16 == 0.  The singular system's left
 * null vector still comes through smpm_batch_set_nullspace. */
int smpm_batch_set_fdm(smpm_batch* b, int npairs, const double* T, const double* T_inv, const smpm_strip_factors* f);
/* b_S = B (A - mu)^{-1} f per system; f: device, nsys x r (r = m_x m_z n^2, reference node order
 * ((ex m_z + ez) n + ix) n + iz, proj/src/mesh.cpp:27-40); b_S: device nsys x k */
int smpm_schur_rhs(smpm_batch* b, const double* f, double* b_S, void* stream);             /* proj/src/schur.cpp:182-186 */
/* u = (A - mu)^{-1} (f - E x_S) per system; f, u: device nsys x r; x_S: device nsys x k */
int smpm_recover_solution(smpm_batch* b, const double* f, const double* x_S, double* u,
                          void* stream);                                                    /* proj/src/schur.cpp:227-230 */

/* ---- transverse Fourier transforms of the 3D extension ----
 * field: device, r x m_y column-major (plane y = field + y r); coeff: device,
 * m_y x r = (m_y / 2) modes x (real, imaginary) as Schur-batch systems 2 j + part.
 * m_y a power of two in [2, 4096]. */
int smpm_fourier_y(long long r, int m_y, const double* field, double* coeff, void* stream);         /* proj/src/fourier.cpp:47-62 */
int smpm_inverse_fourier_y(long long r, int m_y, const double* coeff, double* field, void* stream); /* proj/src/fourier.cpp:64-86 */

/* ---- solves --------------------------------------------------------------- */
/* Batched solve of S x_S = b_S for every system of the batch with `method`
 * (dbj: proj/src/deflation.cpp:102-122, 2las: :124-143, bj: proj/src/gmres.cpp:144-150,
 * schur: proj/src/solver.cpp:56-64). b_S, x_S: device, nsys x k. reports: host,
 * nsys entries (nullable). history: host, nsys x (max_iter + 2) (nullable). */
int smpm_solve(smpm_batch* b, int method, const double* b_S, double* x_S, const smpm_solve_options* opt,
               smpm_report* reports, double* history, void* stream);
int smpm_deflated_solve(smpm_batch* b, const double* b_S, double* x_S, const smpm_solve_options* opt,
                        smpm_report* reports, double* history, void* stream);
int smpm_two_level_schwarz_solve(smpm_batch* b, const double* b_S, double* x_S, const smpm_solve_options* opt,
                                 smpm_report* reports, double* history, void* stream);
/* Stacked solve (proj/src/helmholtz.cpp:187-246, the reference bench's 3D
 * default): ONE GMRES whose Krylov vectors are the concatenation of the nsys
 * systems (dbj: right-hand side P_j b_j, operator block-diagonal P_j S_j M_j^{-1};
 * 2las: S_j (M_j^{-1} + Z C_j^{-1} Z^T)), abs tolerance tol * sqrt(sum_j ||b_j||^2);
 * x_S per system as in smpm_solve.  One report (shared by all systems); history:
 * host, max_iter + 2 (nullable).  CGS2, fused deflation, restart <= 126. */
int smpm_solve_stacked(smpm_batch* b, int method, const double* b_S, double* x_S, const smpm_solve_options* opt,
                       smpm_report* report, double* history, void* stream);
/* Stacked solve across GPUs: the stack's systems (Fourier modes) are spread over
 * ranks, each rank holding its own batch; every inner product of the stacked
 * GMRES (proj/src/helmholtz.cpp:187-246: norms, the two CGS2 reductions, the
 * Arnoldi norm) is summed over the local systems and then over the ranks by
 * `fn(user, device_buf, count, stream)`: an in-place sum all-reduce of `count`
 * doubles at `device_buf`, ordered on `stream` (ncclAllReduce(buf, buf, count,
 * ncclDouble, ncclSum, comm, stream) in a C++ caller).  It
 * must return 0 and leave bitwise-identical results on every rank (NCCL does),
 * so all ranks take the same stopping decisions.  fn = NULL: single rank. */
typedef int (*smpm_allreduce_fn)(void* user, double* device_buf, int count, void* stream);
int smpm_batch_set_allreduce(smpm_batch* b, smpm_allreduce_fn fn, void* user);
/* Same as smpm_solve with HOST b_S / x_S: the H2D and D2H copies are inside
 * the call (the reference-facing end-to-end path). */
int smpm_solve_host(smpm_batch* b, int method, const double* b_S_host, double* x_S_host,
                    const smpm_solve_options* opt, smpm_report* reports, double* history);
/* Starts the host -> device copy of a right-hand-side array (nsys x k, ideally
 * pinned) on a side stream and returns at once; a later smpm_solve_host with the
 * SAME host pointer uses that upload instead of copying.  Called for the next
 * batch before the current smpm_solve_host, it hides the upload behind the
 * current solve (two uploads may be outstanding; the host buffer must stay
 * unchanged until its solve has started).  No reference counterpart: the
 * reference's solve_3d is host-resident. */
int smpm_prefetch_rhs(smpm_batch* b, const double* b_S_host);

/* Number of kernels this library launched since the batch was created
 * (instrumentation for bench.py's gpu_launches). */
long long smpm_batch_launch_count(const smpm_batch* b);

/* Optional device timing of kernel classes (0 Schur GEMM, 1 block-Jacobi
 * GEMMs, 2 deflation, 3 Arnoldi orthogonalization, 4 other, 5 reserved,
 * 6 grid-persistent tail, 7 spectral per-mode pass, 8 shared-matrix
 * transforms, 9 reserved; nclass <= 10), measured with
 * CUDA events on the launching stream during solves/operators. Reads the
 * accumulated milliseconds/launch counts (nullable), then, if enable >= 0,
 * resets them and turns timing on (1) or off (0). */
int smpm_batch_profile(smpm_batch* b, int enable, double* ms, long long* counts, int nclass);

/* Performance knobs of a batch (no reference counterpart; defaults are the
 * measured-best settings). Keys: segb, spec_v2, xform, sp_stage, spectral, spec_2las,
 * p2fuse, cgs_defer, cgs_lanes, xform_parity, gt_vblock, grid_per_sm, gt_ctas, coarse_fork, grid_nocoop (profilers only: the
 * tail then launches without the co-residency guarantee of a cooperative
 * launch), pdl, pythag, grid, grid_max, tail_rows (the tail runs only while
 * live systems x k <= tail_rows; default 200000), post_fuse, early; with b = NULL:
 * fy_tile (transverse FFT). SMPM_EINVAL for an unknown key. The library reads
 * no environment variables. */
int smpm_batch_set_tuning(smpm_batch* b, const char* key, long long value);
/* Which kernels a finalized batch runs (instrumentation for bench.py's work
 * accounting). Keys: xform_kernel (0 tiled contraction plan, 1 resident-slice
 * transform, 2 K-streamed transform, 3 parity-split transform), xform_parity
 * (1 when T is parity-pure and the transforms run as two half-size
 * contractions), cgs_defer (1 when the deferred CGS2 passes apply to fused dbj
 * solves), spectral (1 when the spectral operator form is active). */
int smpm_batch_query(const smpm_batch* b, const char* key, long long* value);
/* Phase-trace dump of the grid-persistent tail into `path` (appended; NULL or
 * "" off): which = 0 per-step phase timestamps, 1 per-CTA timestamps. */
int smpm_batch_set_trace(smpm_batch* b, int which, const char* path);

/* Measured fp64 throughput of the device (TFLOP/s): FP64 FMA pipe and the
 * legacy fp64 tensor-core mma.sync (no tcgen05 f64 kind exists). Roofline
 * denominator for the fp64 contractions. */
int smpm_fp64_peak(int device, double* dfma_tflops, double* dmma_tflops);

#ifdef __cplusplus
}
#endif

#endif /* SMPM_B200_H */
