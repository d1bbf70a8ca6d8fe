// Shared-memory 128-bit access patterns: wavefronts per warp instruction (read with ncu
// --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum).
#include <cstdio>
__device__ __forceinline__ int unit_of(int P, int l) {
  switch (P) {
    case 0: return l;                         // contiguous 512 B
    case 1: return l + (l >> 3);              // padded k + k/8
    case 2: return (l & 7) * 577 + (l >> 3);  // 8 fibres, 577-unit buffers (fibre-fast lanes)
    case 3: return 9 * l;                     // stride 9 units
    case 4: return l * 145;                   // one lane per 145-unit buffer
    case 5: return (l >> 3) * 577 + (l & 7);  // 4 buffers, 8 contiguous each
    case 6: return (l & 15) + (l >> 4) * 32;  // two 256 B halves 512 B apart
    case 7: return 2 * l;                     // stride 2 units (32 B)
  }
  return l;
}
template <int P>
__global__ void k(double2* out, int reps) {
  extern __shared__ double2 s[];
  for (int i = threadIdx.x; i < 8 * 577 + 64; i += blockDim.x) s[i] = make_double2(i, i);
  __syncthreads();
  const int u = unit_of(P, threadIdx.x & 31) + ((threadIdx.x >> 5) & 1) * 0;
  double2 acc = make_double2(0, 0);
  for (int r = 0; r < reps; ++r) {
    double2 v = s[u];
    acc.x += v.x; acc.y += v.y;
    asm volatile("" ::: "memory");
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double2* out; cudaMalloc(&out, 1 << 20);
  const int smem = (8 * 577 + 64) * 16;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<0><<<1, 32, smem>>>(out, 100); k<1><<<1, 32, smem>>>(out, 100); k<2><<<1, 32, smem>>>(out, 100);
  k<3><<<1, 32, smem>>>(out, 100); k<4><<<1, 32, smem>>>(out, 100); k<5><<<1, 32, smem>>>(out, 100);
  k<6><<<1, 32, smem>>>(out, 100); k<7><<<1, 32, smem>>>(out, 100);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
}
