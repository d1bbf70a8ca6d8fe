// Shared helpers for libfftlasso_b200 (sm_100a): status codes, error capture,
// round-to-nearest arithmetic wrappers that forbid FMA contraction, and
// deterministic block reductions.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/fftlasso_b200.h"

namespace fl {

// ---- error state (thread-local message, returned through fl_last_error) ----
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define FL_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t err__ = (call);                                                    \
    if (err__ != cudaSuccess)                                                      \
      return ::fl::fail(FL_E_CUDA, std::string(#call ": ") + cudaGetErrorString(err__)); \
  } while (0)

#define FL_LAUNCH_CHECK() FL_CUDA(cudaGetLastError())

#define FL_TRY(expr)        \
  do {                      \
    int st__ = (expr);      \
    if (st__ != FL_OK) return st__; \
  } while (0)

// ---- exact IEEE ops in NumPy's evaluation order (no FMA contraction) ----
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

// ---- reductions: warp shuffles, then a fixed-order smem tree ----
template <class Op>
__device__ __forceinline__ double warp_reduce(double v, Op op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

struct SumOp {
  static constexpr double identity = 0.0;
  __device__ double operator()(double a, double b) const { return a + b; }
};
struct MaxOp {
  static constexpr double identity = -__builtin_huge_val();
  __device__ double operator()(double a, double b) const { return fmax(a, b); }
};
struct MinOp {
  static constexpr double identity = __builtin_huge_val();
  __device__ double operator()(double a, double b) const { return fmin(a, b); }
};
// NaN-propagating max / min (np.max / np.min semantics) for the final combine.
struct PropMaxOp {
  static constexpr double identity = -__builtin_huge_val();
  __device__ double operator()(double a, double b) const { return (a != a || b != b) ? a + b : fmax(a, b); }
};
struct PropMinOp {
  static constexpr double identity = __builtin_huge_val();
  __device__ double operator()(double a, double b) const { return (a != a || b != b) ? a + b : fmin(a, b); }
};

// Reduce one value per thread to thread 0 of the block.  ``red`` must hold
// 32 doubles.  Deterministic: the combine order depends only on blockDim.
template <class Op>
__device__ __forceinline__ double block_reduce(double v, Op op, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_reduce(v, op);
  __syncthreads();  // protect ``red`` against a previous use
  if (lane == 0) red[warp] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  if (warp == 0) {
    v = lane < nw ? red[lane] : Op::identity;
    v = warp_reduce(v, op);
  }
  return v;  // valid in thread 0
}

// Partial-slot layout: the kernels that reduce write ``K`` scalars per block
// to ``partials[k * gridDim.x + blockIdx.x]``; finish_reduce combines each row
// in block order.
enum RedKind : int { RED_SUM = 0, RED_MAX = 1, RED_MIN = 2 };

// Host-side helpers implemented in fl_runtime.cu
struct Scratch {
  double* partials = nullptr;  // device, kPartialSlots doubles
  double* result = nullptr;    // device, kResultSlots doubles
  double* host = nullptr;      // pinned host mirror of ``result``
};
constexpr int kPartialSlots = 1 << 20;
constexpr int kResultSlots = 64;
constexpr int kMaxRedBlocks = 1184;  // 148 SMs x 8

int scratch(Scratch** out);
// Combine ``nk`` rows of ``nblocks`` partials into result[slot0 + k] with the
// given kinds, on ``stream``.
int finish_reduce(const double* partials, int nblocks, int nk, const int* kinds,
                  double* result, cudaStream_t stream);
// Copy ``count`` result slots to the pinned host mirror and wait.
int fetch_results(Scratch* s, int count, cudaStream_t stream);

inline int grid_for(int64_t n, int threads, int cap = kMaxRedBlocks) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)(b < cap ? b : cap);
}

}  // namespace fl
