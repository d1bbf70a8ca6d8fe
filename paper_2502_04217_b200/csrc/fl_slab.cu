// Slab transposes for the sharded 3D transform (row e of SURVEY 8).
//
// Grid (d0, d1, d2), P ranks, d0 = P a, d1 = P b.  X-slab (a, d1, d2): axes 1
// and 2 local.  Y-slab (b, d2, d0): axis 0 local AND contiguous, so the fused
// synth / mask / analysis pass of fl_fastpass.cu runs on it unchanged.  The
// all-to-all moves P blocks of (a, b, d2) per rank; these kernels build and
// consume those blocks.  X-side kernels are contiguous runs of d2 (16-byte
// moves); Y-side kernels transpose (i0, i2) through 32x33 shared tiles.
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "fl_common.cuh"
#include "fl_internal.h"

namespace fl {
namespace {

constexpr int T = 256;

// send[s][i0][j1][i2] = x[i0][s b + j1][i2]   (PACK = true)
// x[i0][s b + j1][i2] = recv[s][i0][j1][i2]   (PACK = false)
template <bool PACK>
__global__ void k_x_blocks(int64_t a, int64_t d1, int64_t d2h, int P, const double2* __restrict__ src,
                           double2* __restrict__ dst) {
  const int64_t b = d1 / P;
  const int64_t total = a * d1 * d2h;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    // o indexes the block layout (s, i0, j1, i2h)
    const int64_t i2 = o % d2h;
    int64_t t = o / d2h;
    const int64_t j1 = t % b;
    t /= b;
    const int64_t i0 = t % a;
    const int64_t s = t / a;
    const int64_t xi = (i0 * d1 + s * b + j1) * d2h + i2;
    if (PACK) dst[o] = src[xi];
    else dst[xi] = src[o];
  }
}

// Y-slab <-> blocks: y[j1][i2][r a + i0] <-> blk[r][i0][j1][i2].
// One CTA per (r, j1, 32x32 tile of (i0, i2)); smem tile padded to 33.
template <bool TO_Y>
__global__ void k_y_blocks(int64_t a, int64_t b, int64_t d2, int P, const double* __restrict__ src,
                           double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int64_t d0 = a * P;
  const int64_t t0 = (a + 31) / 32, t2 = (d2 + 31) / 32;
  int64_t id = blockIdx.x;
  const int64_t ti2 = id % t2;
  id /= t2;
  const int64_t ti0 = id % t0;
  id /= t0;
  const int64_t j1 = id % b;
  const int64_t r = id / b;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  const int64_t base0 = ti0 * 32, base2 = ti2 * 32;
  if (TO_Y) {
    // read blocks: i2 fastest (tx), i0 rows (ty)
    for (int k = ty; k < 32; k += 8) {
      const int64_t i0 = base0 + k, i2 = base2 + tx;
      if (i0 < a && i2 < d2) tile[k][tx] = src[((r * a + i0) * b + j1) * d2 + i2];
    }
    __syncthreads();
    // write y: i0 fastest (tx), i2 rows (ty)
    for (int k = ty; k < 32; k += 8) {
      const int64_t i2 = base2 + k, i0 = base0 + tx;
      if (i0 < a && i2 < d2) dst[(j1 * d2 + i2) * d0 + r * a + i0] = tile[tx][k];
    }
  } else {
    for (int k = ty; k < 32; k += 8) {
      const int64_t i2 = base2 + k, i0 = base0 + tx;
      if (i0 < a && i2 < d2) tile[tx][k] = src[(j1 * d2 + i2) * d0 + r * a + i0];
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
      const int64_t i0 = base0 + k, i2 = base2 + tx;
      if (i0 < a && i2 < d2) dst[((r * a + i0) * b + j1) * d2 + i2] = tile[k][tx];
    }
  }
}

// ---- fused exchange over peer memory -----------------------------------
// One kernel per direction replaces pack -> all-to-all -> unpack: every
// element is read once from the local slab and stored once, transposed, into
// its final place in the OWNING rank's slab (a peer pointer over NVLink /
// NVSwitch for remote ranks, the local buffer for this rank).  The 32x33
// shared tile turns the layout change into 256-byte coalesced row stores on
// both sides.
//
// Ordering: the stores to peer slabs must be visible on the owning GPU before
// it reads them.  Each CTA ends with a barrier and one system-scope fence
// (cumulative over the CTA's stores, which the barrier ordered before it);
// the caller then puts a stream-ordered cross-rank barrier (a one-element
// NCCL all-reduce) between this kernel and the first read on the peer.
//
// The destination table (one slab pointer per rank) lives in device memory
// (uploaded once per distinct table, see peer_table) and is read with a
// uniform or per-thread global load -- no by-value pointer array indexed
// dynamically (that forces a local-memory copy of the parameter block).
constexpr int kMaxPeers = 16;

__device__ __forceinline__ void publish_system() {
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

// X-slab (a, d1, d2) of rank `me` -> Y-slabs (b, d2, d0) of every rank:
//   Y[j / b][((j % b) d2 + i2) d0 + me a + i0] = x[(i0 d1 + j) d2 + i2]
// One CTA per (j, 32x32 tile of (i0, i2)).
// (ac planes starting at plane i0off of the slab: the chunked, overlapped form)
__global__ void k_x_to_y_peers(int64_t a, int64_t d1, int64_t d2, int P, int me, const double* __restrict__ x,
                               double* const* __restrict__ dst, int64_t ac, int64_t i0off) {
  __shared__ double tile[32][33];
  const int64_t b = d1 / P, d0 = a * P;
  const int64_t t0 = (ac + 31) / 32, t2 = (d2 + 31) / 32;
  int64_t id = blockIdx.x;
  const int64_t ti2 = id % t2;
  id /= t2;
  const int64_t ti0 = id % t0;
  const int64_t j = id / t0;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t base0 = ti0 * 32, base2 = ti2 * 32;
  for (int k = ty; k < 32; k += 8) {  // read: i2 fastest
    const int64_t i0 = base0 + k, i2 = base2 + tx;
    if (i0 < ac && i2 < d2) tile[k][tx] = x[(i0 * d1 + j) * d2 + i2];
  }
  __syncthreads();
  double* y = dst[j / b];
  const int64_t j1 = j % b;
  for (int k = ty; k < 32; k += 8) {  // write: i0 fastest
    const int64_t i2 = base2 + k, i0 = base0 + tx;
    if (i0 < ac && i2 < d2) y[(j1 * d2 + i2) * d0 + me * a + i0off + i0] = tile[tx][k];
  }
  publish_system();
}

// Y-slab (b, d2, d0) of rank `me` -> X-slabs (a, d1, d2) of every rank:
//   X[i / a][((i % a) d1 + me b + j1) d2 + i2] = y[(j1 d2 + i2) d0 + i]
// One CTA per (j1, 32x32 tile of (i, i2)).
__global__ void k_y_to_x_peers(int64_t a, int64_t b, int64_t d2, int P, int me, const double* __restrict__ y,
                               double* const* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int64_t d0 = a * P, d1 = b * P;
  const int64_t ti_n = (d0 + 31) / 32, t2 = (d2 + 31) / 32;
  int64_t id = blockIdx.x;
  const int64_t ti2 = id % t2;
  id /= t2;
  const int64_t ti = id % ti_n;
  const int64_t j1 = id / ti_n;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t base = ti * 32, base2 = ti2 * 32;
  for (int k = ty; k < 32; k += 8) {  // read: i fastest
    const int64_t i2 = base2 + k, i = base + tx;
    if (i < d0 && i2 < d2) tile[tx][k] = y[(j1 * d2 + i2) * d0 + i];
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {  // write: i2 fastest
    const int64_t i = base + k, i2 = base2 + tx;
    if (i < d0 && i2 < d2) dst[i / a][((i % a) * d1 + me * b + j1) * d2 + i2] = tile[k][tx];
  }
  publish_system();
}

// Device copy of a host pointer table, cached per (device, table contents):
// a grid's exchange tables are fixed for its lifetime, so each is uploaded
// once.  Bounded: past kMaxTables distinct tables the cache is dropped after
// a device synchronisation (no in-flight exchange can still read a table).
int peer_table(int P, double* const* ptrs, double* const** out) {
  if (P < 1 || P > kMaxPeers) return fail(FL_E_VALUE, "peer exchange supports 1..16 ranks");
  int dev = 0;
  FL_CUDA(cudaGetDevice(&dev));
  std::vector<uintptr_t> key(1, (uintptr_t)dev);
  for (int r = 0; r < P; ++r) {
    if (!ptrs[r]) return fail(FL_E_VALUE, "null peer pointer");
    key.push_back((uintptr_t)ptrs[r]);
  }
  static std::mutex mu;
  static std::map<std::vector<uintptr_t>, double**> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  constexpr size_t kMaxTables = 256;
  if (it == cache.end() && cache.size() >= kMaxTables) {
    for (auto& kv : cache) {  // each table's device: finish its work, then free
      cudaSetDevice((int)kv.first[0]);
      cudaDeviceSynchronize();
      cudaFree(kv.second);
    }
    FL_CUDA(cudaSetDevice(dev));
    cache.clear();
  }
  if (it == cache.end()) {
    double** d = nullptr;
    FL_CUDA(cudaMalloc(&d, sizeof(double*) * P));
    FL_CUDA(cudaMemcpy(d, ptrs, sizeof(double*) * P, cudaMemcpyHostToDevice));
    it = cache.emplace(key, d).first;
  }
  *out = it->second;
  return FL_OK;
}

int x_blocks(bool pack, int64_t a, int64_t d1, int64_t d2, int P, const double* src, double* dst,
             cudaStream_t s) {
  if (P < 1 || d1 % P || d2 % 2) return fail(FL_E_SHAPE, "slab transpose needs d1 % P == 0 and even d2");
  const int64_t total = a * d1 * (d2 / 2);
  const int grid = (int)std::min<int64_t>((total + T - 1) / T, 148 * 16);
  if (pack) k_x_blocks<true><<<grid, T, 0, s>>>(a, d1, d2 / 2, P, (const double2*)src, (double2*)dst);
  else k_x_blocks<false><<<grid, T, 0, s>>>(a, d1, d2 / 2, P, (const double2*)src, (double2*)dst);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int y_blocks(bool to_y, int64_t a, int64_t b, int64_t d2, int P, const double* src, double* dst,
             cudaStream_t s) {
  if (P < 1) return fail(FL_E_SHAPE, "bad rank count");
  const int64_t blocks = (int64_t)P * b * ((a + 31) / 32) * ((d2 + 31) / 32);
  if (blocks > 0x7fffffffLL) return fail(FL_E_SHAPE, "slab too large");
  if (to_y) k_y_blocks<true><<<(unsigned)blocks, T, 0, s>>>(a, b, d2, P, src, dst);
  else k_y_blocks<false><<<(unsigned)blocks, T, 0, s>>>(a, b, d2, P, src, dst);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

}  // namespace
}  // namespace fl

using namespace fl;

extern "C" {

int fl_slab_pack_x(int64_t a, int64_t d1, int64_t d2, int nranks, const double* x_slab, double* send,
                   fl_stream_t stream) {
  if (!x_slab || !send) return fail(FL_E_VALUE, "null argument");
  return x_blocks(true, a, d1, d2, nranks, x_slab, send, (cudaStream_t)stream);
}

int fl_slab_unpack_x(int64_t a, int64_t d1, int64_t d2, int nranks, const double* recv, double* x_slab,
                     fl_stream_t stream) {
  if (!x_slab || !recv) return fail(FL_E_VALUE, "null argument");
  return x_blocks(false, a, d1, d2, nranks, recv, x_slab, (cudaStream_t)stream);
}

int fl_slab_unpack_y(int64_t a, int64_t b, int64_t d2, int nranks, const double* recv, double* y_slab,
                     fl_stream_t stream) {
  if (!y_slab || !recv) return fail(FL_E_VALUE, "null argument");
  return y_blocks(true, a, b, d2, nranks, recv, y_slab, (cudaStream_t)stream);
}

int fl_slab_pack_y(int64_t a, int64_t b, int64_t d2, int nranks, const double* y_slab, double* send,
                   fl_stream_t stream) {
  if (!y_slab || !send) return fail(FL_E_VALUE, "null argument");
  return y_blocks(false, a, b, d2, nranks, y_slab, send, (cudaStream_t)stream);
}

int fl_slab_x_to_y_peers_planes(int64_t a, int64_t d1, int64_t d2, int nranks, int rank, int64_t i0_begin,
                                int64_t i0_count, const double* x_planes, double* const* y_slabs,
                                fl_stream_t stream) {
  if (!x_planes || !y_slabs) return fail(FL_E_VALUE, "null argument");
  if (nranks < 1 || d1 % nranks || rank < 0 || rank >= nranks) return fail(FL_E_SHAPE, "bad slab geometry");
  if (i0_begin < 0 || i0_count < 0 || i0_begin + i0_count > a) return fail(FL_E_SHAPE, "plane range outside the slab");
  double* const* pe = nullptr;
  FL_TRY(peer_table(nranks, y_slabs, &pe));
  const int64_t blocks = d1 * ((i0_count + 31) / 32) * ((d2 + 31) / 32);
  if (blocks > 0x7fffffffLL) return fail(FL_E_SHAPE, "slab too large");
  if (blocks == 0) return FL_OK;
  k_x_to_y_peers<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(a, d1, d2, nranks, rank, x_planes, pe,
                                                                       i0_count, i0_begin);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fl_slab_x_to_y_peers(int64_t a, int64_t d1, int64_t d2, int nranks, int rank, const double* x_slab,
                         double* const* y_slabs, fl_stream_t stream) {
  return fl_slab_x_to_y_peers_planes(a, d1, d2, nranks, rank, 0, a, x_slab, y_slabs, stream);
}

int fl_slab_y_to_x_peers(int64_t a, int64_t b, int64_t d2, int nranks, int rank, const double* y_slab,
                         double* const* x_slabs, fl_stream_t stream) {
  if (!y_slab || !x_slabs) return fail(FL_E_VALUE, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(FL_E_SHAPE, "bad slab geometry");
  double* const* pe = nullptr;
  FL_TRY(peer_table(nranks, x_slabs, &pe));
  const int64_t blocks = b * ((a * nranks + 31) / 32) * ((d2 + 31) / 32);
  if (blocks > 0x7fffffffLL) return fail(FL_E_SHAPE, "slab too large");
  if (blocks == 0) return FL_OK;
  k_y_to_x_peers<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(a, b, d2, nranks, rank, y_slab, pe);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

// Device buffers shareable across processes (cudaMalloc'd, so an IPC handle
// names exactly this allocation) for the peer exchange.
int fl_ipc_alloc(int64_t bytes, void** ptr, unsigned char* handle64) {
  if (!ptr || !handle64 || bytes <= 0) return fail(FL_E_VALUE, "bad argument");
  FL_CUDA(cudaMalloc(ptr, (size_t)bytes));
  cudaIpcMemHandle_t h;
  FL_CUDA(cudaIpcGetMemHandle(&h, *ptr));
  static_assert(sizeof(h) == 64, "IPC handle is 64 bytes");
  memcpy(handle64, &h, 64);
  return FL_OK;
}

int fl_ipc_open(const unsigned char* handle64, void** ptr) {
  if (!ptr || !handle64) return fail(FL_E_VALUE, "bad argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  FL_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return FL_OK;
}

int fl_ipc_close(void* ptr) {
  if (ptr) FL_CUDA(cudaIpcCloseMemHandle(ptr));
  return FL_OK;
}

int fl_dev_free(void* ptr) {
  if (ptr) FL_CUDA(cudaFree(ptr));
  return FL_OK;
}

}  // extern "C"
