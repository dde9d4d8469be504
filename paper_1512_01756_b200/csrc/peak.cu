// fp64 throughput microbenchmarks (sm_100a): the roofline denominator for the
// fp64 contractions, since MEASURED_PEAKS.json carries no fp64 figure.
//  - DFMA: independent FMA chains on the FP64 pipe
//  - DMMA: legacy fp64 tensor-core mma.sync.m8n8k4 (tcgen05 has no f64 kind)
#include <cuda_runtime.h>

#include <string>

#include "../../include/smpm_b200.h"

namespace {

constexpr int kChains = 16;

__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double b, double c) {
  double a[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  if (s == 1234.5678) out[blockIdx.x] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double a = 1e-3 * threadIdx.x, bb = 1e-3 * (threadIdx.x + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1])
                   : "d"(a), "d"(bb));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1234.5678) out[blockIdx.x] = s;
}

}  // namespace

extern "C" int smpm_fp64_peak(int device, double* dfma_tflops, double* dmma_tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return SMPM_ECUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return SMPM_ECUDA;
  const int blocks = prop.multiProcessorCount * 8, threads = 256;
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double) * blocks) != cudaSuccess) return SMPM_ECUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time_it = [&](auto launch, double flops) {
    launch();  // warm-up
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    return 3.0 * flops / (ms * 1e-3) / 1e12;
  };
  const int it1 = 4096, it2 = 2048;
  const double f1 = 2.0 * kChains * double(it1) * blocks * threads;
  const double f2 = 2.0 * 256.0 * 8 * double(it2) * blocks * (threads / 32);
  const double t1 = time_it([&] { dfma_peak_kernel<<<blocks, threads>>>(out, it1, 0.999999, 1e-7); }, f1);
  const double t2 = time_it([&] { dmma_peak_kernel<<<blocks, threads>>>(out, it2); }, f2);
  const cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err != cudaSuccess) return SMPM_ECUDA;
  if (dfma_tflops) *dfma_tflops = t1;
  if (dmma_tflops) *dmma_tflops = t2;
  return SMPM_OK;
}
