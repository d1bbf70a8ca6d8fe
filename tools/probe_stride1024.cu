// DRAM access-pattern probe for the strided passes at 1024^3 (fp64): copy the
// grid tile by tile, a tile = SEG contiguous bytes of each of the 1024 rows of
// an axis (axis 0: rows 8 MiB apart; axis 1: rows 8 KiB apart), each thread
// holding 8 16-byte elements between its loads and stores.  Shows the copy
// floor of the tile shapes the m = 1024 strided engines use (E = 16 engine:
// 64-byte segments; split engine: 128-byte segments) against wider ones.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_stride1024 tools/probe_stride1024.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr long long M = 1024;

// axis 0: tile t = segment of plane-row (i1), rows i0 = 0..M-1 at stride M*M
// axis 1: tile t = segment of (i0, i2-range), rows i1 = 0..M-1 at stride M
template <int SEG, int T, int AXIS>
__global__ void __launch_bounds__(T) copy_tiles(const double2* __restrict__ x, double2* __restrict__ y,
                                                long long ntiles) {
  constexpr int LANES = SEG / 16;
  constexpr int ROWS_PER_PASS = T / LANES;
  constexpr int E = 8;
  constexpr long long SEGS = (M * 8 / 16) / LANES;                      // segments per contiguous row
  constexpr long long RSTRIDE = AXIS == 0 ? (M * M / 2) : (M / 2);      // row stride in double2
  const int lane = threadIdx.x % LANES, r0 = threadIdx.x / LANES;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long outer = t / SEGS, seg = t % SEGS;
    const long long base = (AXIS == 0 ? outer * (M / 2) : outer * (M * M / 2)) + seg * LANES + lane;
    for (int r = r0; r < M; r += ROWS_PER_PASS * E) {
      double2 v[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int row = r + e * ROWS_PER_PASS;
        v[e] = row < M ? x[base + row * RSTRIDE] : make_double2(0, 0);
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int row = r + e * ROWS_PER_PASS;
        if (row < M) y[base + row * RSTRIDE] = v[e];
      }
    }
  }
}

template <int SEG, int T, int AXIS>
void run(double2* x, double2* y, int per_sm) {
  const long long ntiles = M * ((M * 8 / 16) / (SEG / 16));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = 148 * per_sm;
  copy_tiles<SEG, T, AXIS><<<grid, T>>>(x, y, ntiles);
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) copy_tiles<SEG, T, AXIS><<<grid, T>>>(x, y, ntiles);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double gbs = 2.0 * 16.0 * M * M * M / 2 / (ms * 1e6);
  printf("axis-%d tile copy  SEG %5d B  %4d thr  %d CTA/SM  %8.3f ms  %7.0f GB/s\n", AXIS, SEG, T, per_sm, ms, gbs);
}

int main() {
  double2 *x, *y;
  const size_t bytes = (size_t)M * M * M * 8;
  if (cudaMalloc(&x, bytes) != cudaSuccess || cudaMalloc(&y, bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(x, 0, bytes);
  run<64, 256, 0>(x, y, 8);
  run<128, 256, 0>(x, y, 8);
  run<256, 256, 0>(x, y, 8);
  run<512, 256, 0>(x, y, 8);
  run<64, 256, 1>(x, y, 8);
  run<128, 256, 1>(x, y, 8);
  run<256, 256, 1>(x, y, 8);
  run<512, 256, 1>(x, y, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaMemcpy(y, x, bytes, cudaMemcpyDeviceToDevice);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("cudaMemcpy D2D (contiguous)                      %8.3f ms  %7.0f GB/s\n", ms, 2.0 * bytes / (ms * 1e6));
  return 0;
}
