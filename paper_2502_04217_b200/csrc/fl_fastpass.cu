// Dispatcher of the register-resident pass kernels (templates in
// fl_fastpass.cuh).  The per-length instantiations live in fl_fp_small.cu,
// fl_fp_512.cu and fl_fp_large.cu so they compile in parallel.
#include <cstdlib>

#include "fl_fastpass.cuh"

namespace fl {
namespace fpk {

Entry make_16(bool strided, int kind, bool epi);
Entry make_32(bool strided, int kind, bool epi);
Entry make_64(bool strided, int kind, bool epi);
Entry make_128(bool strided, int kind, bool epi);
Entry make_256(bool strided, int kind, bool epi);
Entry make_512(bool strided, int kind, bool epi);
Entry make_1024(bool strided, int kind, bool epi);
Entry make_2048(bool strided, int kind, bool epi);
Entry make_4096(bool strided, int kind, bool epi);
Entry make_8192(bool strided, int kind, bool epi);
Entry make_mirror_1024(int kind);
Entry make_group_512(int kind, bool epi);
Entry make_warp_1024(int kind, bool epi, bool nrm);
Entry make_group_2048(int kind, bool epi);

Entry lookup(int m, bool strided, int kind, bool epi) {
  switch (m) {
    case 16: return make_16(strided, kind, epi);
    case 32: return make_32(strided, kind, epi);
    case 64: return make_64(strided, kind, epi);
    case 128: return make_128(strided, kind, epi);
    case 256: return make_256(strided, kind, epi);
    case 512: return make_512(strided, kind, epi);
    case 1024: return make_1024(strided, kind, epi);
    case 2048: return make_2048(strided, kind, epi);
    case 4096: return make_4096(strided, kind, epi);
    case 8192: return make_8192(strided, kind, epi);
    default: return Entry();
  }
}

// Called once per (device, kernel): the shared-memory opt-in is a per-device
// function attribute.
int grid_of(Entry& e, int* out) {
  int dev = 0, sms = 0;
  FL_CUDA(cudaGetDevice(&dev));
  FL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaFuncAttributes fa;
  FL_CUDA(cudaFuncGetAttributes(&fa, e.fn));
  FL_CUDA(cudaFuncSetAttribute(e.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               227 * 1024 - (int)fa.sharedSizeBytes));
  int per_sm = 0;
  FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, e.fn, e.threads, e.smem));
  if (per_sm < 1) return fail(FL_E_CUDA, "fast pass kernel cannot be resident");
  *out = per_sm * sms;
  return FL_OK;
}

}  // namespace fpk

using fpk::Entry;
using fpk::lookup;
using fpk::grid_of;

bool fast_supported(int m) { return m >= 16 && m <= 8192 && (m & (m - 1)) == 0; }

int launch_fast(int m, bool strided, int kind, bool epi, const PassArgs& A, int* nblocks,
                cudaStream_t s) {
  // persistent grid size per kernel variant (resident CTAs x SMs)
  // keyed by (device, kernel): attributes and SM counts are per device
  static std::mutex mu;
  static std::unordered_map<const void*, int> grids[kMaxDevices];
  // strided m = 1024 synthesis / analysis: the mirrored 8 x 16 x 8 engine
  // (fl_mirror.cuh fft1024; 512-thread CTAs, 128-byte row segments): 1024^3
  // axis 0 6.40 / 6.19 -> 4.93 / 5.23 ms and axis 1 4.98 / 5.58 -> 4.78 / 4.87
  // ms against the round-1 split (two mirrored 512-point halves) and E = 16
  // engines; 256-thread CTAs (64-byte segments) were slower on both axes.
  const bool mir = m == 1024 && strided && !epi && (kind == K_SYNTH || kind == K_ANALYZE);
  // contiguous m = 512 / 1024 / 2048: group-decoupled passes (fl_gpass.cuh);
  // they stage rows with TMA, so the row pointers must be 16-byte aligned
  // (an unaligned view falls back to the CTA-tiled engine).
  const bool aligned = (reinterpret_cast<uintptr_t>(A.in) & 15) == 0 &&
                       (kind != K_RESID || (reinterpret_cast<uintptr_t>(A.bhat) & 15) == 0);
  const bool group = !strided && aligned && (m == 512 || m == 2048) && A.G < (1LL << 30);
  // contiguous m = 1024: the two-stage warp-owned passes (fl_wpass.cuh, one
  // exchange per FFT; 1024^3 gram 5.61 -> 4.70 ms).  At m = 512 neither the
  // 32-element form (255 registers: 8 warps per SM, 1.07 ms) nor a 16-element
  // form with a shuffle radix-2 step (0.65 ms) beats the group passes: the
  // fused gram there is FP64-issue bound (~150 M FP64 warp instructions, the
  // FFT's own flop count), not exchange bound.
  const bool warp = !strided && m == 1024;
  Entry e = mir ? fpk::make_mirror_1024(kind)
            : warp ? fpk::make_warp_1024(kind, epi, A.nrm_partials != nullptr)
            : group ? (m == 512 ? fpk::make_group_512(kind, epi) : fpk::make_group_2048(kind, epi))
                    : lookup(m, strided, kind, epi);
  if (!e.fn) return fail(FL_E_VALUE, "no fast kernel for this pass");
  // the strided fused gram addresses a fibre's rows at 32-bit element offsets
  // k * stride from its base (a grid past 2^32 doubles per array does not fit
  // one GPU's IPM workspace anyway)
  if (strided && kind == K_GRAM && (int64_t)(m - 1) * A.inner >= (int64_t(1) << 32))
    return fail(FL_E_SHAPE, "strided fibre spans 2^32 elements or more");
  int grid_cap = 0, dev = 0;
  FL_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(FL_E_VALUE, "device index out of range");
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = grids[dev].find((const void*)e.fn);
    if (it == grids[dev].end()) {
      FL_TRY(grid_of(e, &grid_cap));
      grids[dev][(const void*)e.fn] = grid_cap;
    } else {
      grid_cap = it->second;
    }
  }
  const int64_t tiles = (A.G + e.w - 1) / e.w;
  const int grid = (int)std::min<int64_t>(tiles, grid_cap);
  e.fn<<<grid, e.threads, e.smem, s>>>(A);
  FL_LAUNCH_CHECK();
  if (nblocks) *nblocks = grid;
  return FL_OK;
}

}  // namespace fl
