// DRAM access-pattern probe for the strided axis-0 pass at 512^3 (fp64):
// copy the grid tile by tile, a tile = SEG contiguous bytes of every one of
// the 512 rows 2 MiB apart (the axis-0 fibre pattern), each thread holding
// 8 16-byte elements in registers between its loads and stores (as the FFT
// engine does).  SEG = 128 B is the shipped pass's segment; wider segments
// show how much row-buffer locality the pattern leaves on the table.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_stride tools/probe_stride.cu
//   ./tools/probe_stride
#include <cstdio>
#include <cuda_runtime.h>

constexpr long long M = 512;
constexpr long long PLANE = M * M;  // doubles between consecutive axis-0 rows

template <int SEG, int T>
__global__ void __launch_bounds__(T) copy_tiles(const double2* __restrict__ x, double2* __restrict__ y,
                                                long long ntiles) {
  constexpr int LANES = SEG / 16;          // 16-byte lanes per row segment
  constexpr int ROWS_PER_PASS = T / LANES; // rows covered by one sweep of the CTA
  constexpr int E = 8;                     // elements held per thread per batch
  const int lane = threadIdx.x % LANES, r0 = threadIdx.x / LANES;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    // tile t: segment (t % segs_per_row) of plane-row (t / segs_per_row)
    constexpr long long SEGS = (M * 8 / 16) / LANES;  // segments per contiguous row of the plane
    const long long base = (t / SEGS) * (M / 2) + (t % SEGS) * LANES + lane;  // in double2
    for (int r = r0; r < M; r += ROWS_PER_PASS * E) {
      double2 v[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int row = r + e * ROWS_PER_PASS;
        v[e] = row < M ? x[base + row * (PLANE / 2)] : make_double2(0, 0);
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int row = r + e * ROWS_PER_PASS;
        if (row < M) y[base + row * (PLANE / 2)] = v[e];
      }
    }
  }
}

// Same 128-byte tiles, but CTAs launched in clusters of CL that take
// adjacent tiles and meet at a cluster barrier after every tile, so the CL
// segments of one row are requested together (row-buffer locality without a
// wider tile).
template <int T, int CL>
__global__ void __launch_bounds__(T) copy_tiles_cluster(const double2* __restrict__ x, double2* __restrict__ y,
                                                        long long ntiles) {
  constexpr int LANES = 8, ROWS_PER_PASS = T / LANES, E = 8;
  constexpr long long SEGS = (M * 8 / 16) / LANES;
  const int lane = threadIdx.x % LANES, r0 = threadIdx.x / LANES;
  const long long nrounds = (ntiles + gridDim.x - 1) / gridDim.x;
  for (long long k = 0; k < nrounds; ++k) {
    const long long t = k * gridDim.x + blockIdx.x;
    if (t < ntiles) {
      const long long base = (t / SEGS) * (M / 2) + (t % SEGS) * LANES + lane;
      for (int r = r0; r < M; r += ROWS_PER_PASS * E) {
        double2 v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = x[base + (r + e * ROWS_PER_PASS) * (PLANE / 2)];
#pragma unroll
        for (int e = 0; e < E; ++e) y[base + (r + e * ROWS_PER_PASS) * (PLANE / 2)] = v[e];
      }
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n barrier.cluster.wait.aligned;\n" ::: "memory");
  }
}

template <int T, int CL>
void run_cluster(const double2* x, double2* y, int sms, int per_sm) {
  const long long ntiles = (M * M * 8 / 16) / 8;
  const int grid = per_sm * sms / CL * CL;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(T);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchKernelEx(&cfg, copy_tiles_cluster<T, CL>, (const double2*)x, y, ntiles);
  cudaEventRecord(a);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, copy_tiles_cluster<T, CL>, (const double2*)x, y, ntiles);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  printf("axis-0 tile copy  SEG   128 B  %4d thr  cluster %d (%d CTA/SM req)  %.4f ms  %6.0f GB/s  [%s]\n", T, CL,
         per_sm, ms, 2.0 * M * M * M * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

template <int SEG, int T>
void run(const double2* x, double2* y, int sms) {
  const long long ntiles = (M * M * 8 / 16) / (SEG / 16);  // plane of M*M doubles in SEG-byte tiles
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, copy_tiles<SEG, T>, T, 0);
  const int grid = per_sm * sms;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  copy_tiles<SEG, T><<<grid, T>>>(x, y, ntiles);
  cudaEventRecord(a);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) copy_tiles<SEG, T><<<grid, T>>>(x, y, ntiles);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double bytes = 2.0 * M * M * M * 8;
  printf("axis-0 tile copy  SEG %5d B  %4d thr  %2d CTA/SM  %.4f ms  %6.0f GB/s\n", SEG, T, per_sm, ms,
         bytes / ms / 1e6);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double2 *x, *y;
  const size_t bytes = M * M * M * 8;
  cudaMalloc(&x, bytes);
  cudaMalloc(&y, bytes);
  cudaMemset(x, 0, bytes);
  run<128, 256>(x, y, sms);
  run<256, 256>(x, y, sms);
  run<512, 256>(x, y, sms);
  run<1024, 256>(x, y, sms);
  run<128, 512>(x, y, sms);
  run<256, 512>(x, y, sms);
  run<512, 512>(x, y, sms);
  run_cluster<256, 2>(x, y, sms, 2);
  run_cluster<256, 4>(x, y, sms, 2);
  run_cluster<256, 8>(x, y, sms, 2);
  run_cluster<256, 2>(x, y, sms, 8);
  run_cluster<256, 4>(x, y, sms, 8);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  // contiguous reference
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) cudaMemcpy(y, x, bytes, cudaMemcpyDeviceToDevice);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("cudaMemcpy D2D (contiguous)                          %.4f ms  %6.0f GB/s\n", ms / 20,
         2.0 * bytes / (ms / 20) / 1e6);
  return 0;
}
