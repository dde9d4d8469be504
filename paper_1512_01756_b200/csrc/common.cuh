// Shared device-side types for the B200 Schur-GMRES kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace smpm {

// Symbolic vector buffers an operator reads/writes; resolved per launch from
// a BufTable so one precomputed job list serves every call.
enum BufId : int { BUF_IN = 0, BUF_OUT = 1, BUF_TMP = 2, BUF_TMP2 = 3, BUF_NONE = 4 };

struct BufTable {
  double* p[4];
};

// Strided column view over a batched vector: element (r, c) lives at
//   buf + off + c*cs + r + (r >= split ? soff : 0)
// which expresses the reference's interface-slot permutations
// (/root/reference/proj/src/schur.cpp:113-124) without gathers.
struct View {
  int buf;
  int split;
  long long off;
  long long cs;
  long long soff;
  __host__ __device__ long long at(int r, int c) const {
    return off + static_cast<long long>(c) * cs + r + (r >= split ? soff : 0);
  }
};

// One dense fp64 contraction: out = beta*add + alpha * op(A) * B
struct GemmJob {
  const double* A;  // column-major, or row-major when transA (A^T of a column-major matrix)
  long long lda;
  int transA;
  int M, N, K;
  int sys;  // owning system (active mask)
  int splitk;       // number of K splits (>= 1)
  int ws_off;       // split-K workspace offset (in BM*BN tiles) of this job's first tile
  View b, out, add;
  double alpha, beta;
};

struct GemmTile {
  int job;
  int m0, n0;
  int ks;  // K-split index
};

// Programmatic dependent launch (kernels of one Arnoldi step are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): a kernel first waits for
// the grid before it (all of its memory operations visible), then lets the next
// kernel of the stream start launching so its CTAs are resident when this one
// drains. Both are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

constexpr int GEMM_BM = 128;
constexpr int GEMM_BN = 32;
constexpr int GEMM_BK = 16;
constexpr int GEMM_THREADS = 256;

}  // namespace smpm
