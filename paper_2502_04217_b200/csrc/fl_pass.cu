// Axis passes of the packed real transform pair A / A^T and the fused gram
// (fourier.py:172-235, masking.py:107-118), sm_100a.
//
// Data model.  The real grid is row-major (d0[, d1[, d2]]).  A pass along
// axis ``a`` transforms fibres of length m = dims[a].  Fibres are processed
// in PAIRS as one complex FFT of length m (x + i y), which halves the FFT
// work of a real transform:
//   * strided axes (a < ndim-1): the pair is two neighbouring fibres along
//     the contiguous axis, so (x, y) is one aligned 16-byte double2 load and
//     a warp reads whole 128-byte row segments of a tile;
//   * the contiguous axis (a = ndim-1): the pair is two neighbouring rows
//     (1D: one row, imaginary part zero).
// The reference's per-fibre packing (fourier.py:176-181 unpack, :193-197
// pack) is folded into the load (synthesis) and store (analysis) stages,
// together with the 1/sqrt(m) ortho scaling.  The last-axis synthesis, the
// missing-sample mask and the last-axis analysis run in ONE pass
// (K_GRAM / K_RESID), so a d-dimensional gram is 2d-1 HBM passes; the KKT
// epilogue (newton_system.py:148-152) and the d.Kd partial dot fuse into
// the store of the final pass.  Every pass is in place (a CTA owns its
// fibres), so no scratch vector is needed.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include <mutex>

#include "fl_common.cuh"
#include "fl_internal.h"
#include "fl_passargs.cuh"

namespace fl {

namespace {

constexpr int kThreads = 256;
constexpr int kSmemBudget = 200 * 1024;
constexpr int kMaxGrid = 148 * 16;

// Mapping of a linear work index onto (fibre f, position j) so that the
// global side is coalesced: fibre-fast on strided axes, position-fast on
// the contiguous axis.
template <bool STRIDED>
__device__ __forceinline__ void split(int idx, int F, int len, int& f, int& j) {
  if (STRIDED) { f = idx % F; j = idx / F; }
  else { j = idx % len; f = idx / len; }
}

// ---- load stages ----
template <bool STRIDED>
__device__ void load_packed(const PassArgs& A, double2* buf, int64_t g0, int nf) {
  const int F = A.F, h = A.h, m = A.m;
  for (int idx = threadIdx.x; idx < F * h; idx += blockDim.x) {
    int f, j;
    split<STRIDED>(idx, F, h, f, j);
    double2* fib = buf + f * A.fs;
    if (f >= nf) {
      fib[j] = make_double2(0.0, 0.0);
      fib[j ? m - j : h] = make_double2(0.0, 0.0);
      continue;
    }
    const Geo q = geo<STRIDED>(A, g0 + f);
    const int64_t ia = q.st * (j ? j + 1 : 0), ib = q.st * (j ? j + h : 1);
    double xa, xb, ya = 0.0, yb = 0.0;
    if (STRIDED) {
      const double2 a = *reinterpret_cast<const double2*>(A.in + q.bx + ia);
      const double2 b = *reinterpret_cast<const double2*>(A.in + q.bx + ib);
      xa = a.x; ya = a.y; xb = b.x; yb = b.y;
    } else {
      xa = A.in[q.bx + ia];
      xb = A.in[q.bx + ib];
      if (q.by >= 0) { ya = A.in[q.by + ia]; yb = A.in[q.by + ib]; }
    }
    if (j == 0) {
      fib[0] = make_double2(A.c0 * xa, A.c0 * ya);
      fib[h] = make_double2(A.c0 * xb, A.c0 * yb);
    } else {
      fib[j] = make_double2(A.c1 * (xa - yb), A.c1 * (xb + ya));
      fib[m - j] = make_double2(A.c1 * (xa + yb), A.c1 * (ya - xb));
    }
  }
}

template <bool STRIDED>
__device__ void load_plain(const PassArgs& A, double2* buf, int64_t g0, int nf) {
  const int F = A.F, m = A.m;
  for (int idx = threadIdx.x; idx < F * m; idx += blockDim.x) {
    int f, k;
    split<STRIDED>(idx, F, m, f, k);
    double2 z = make_double2(0.0, 0.0);
    if (f < nf) {
      const Geo q = geo<STRIDED>(A, g0 + f);
      if (STRIDED) z = *reinterpret_cast<const double2*>(A.in + q.bx + k * q.st);
      else {
        z.x = A.in[q.bx + k];
        if (q.by >= 0) z.y = A.in[q.by + k];
      }
    }
    buf[f * A.fs + k] = z;
  }
}

// ---- middle stage of the fused last-axis pass: Z (b_hat - x) or Z x ----
template <bool RESID>
__device__ void apply_mask(const PassArgs& A, double2* buf, int64_t g0, int nf, double& nrm) {
  const int F = A.F, m = A.m;
  for (int idx = threadIdx.x; idx < F * m; idx += blockDim.x) {
    int f, k;
    split<false>(idx, F, m, f, k);
    if (f >= nf) continue;
    const Geo q = geo<false>(A, g0 + f);
    double2 z = buf[f * A.fs + k];
    const int64_t vx = q.bx + k;
    if (RESID) z.x = missing(A.bits, vx) ? 0.0 : A.bhat[vx] - z.x;
    else if (missing(A.bits, vx)) z.x = 0.0;
    if (q.by >= 0) {
      const int64_t vy = q.by + k;
      if (RESID) z.y = missing(A.bits, vy) ? 0.0 : A.bhat[vy] - z.y;
      else if (missing(A.bits, vy)) z.y = 0.0;
    } else {
      z.y = 0.0;
    }
    if (!RESID) nrm += z.x * z.x + z.y * z.y;
    buf[f * A.fs + k] = z;
  }
}

// ---- store stages ----
template <bool STRIDED>
__device__ void store_plain(const PassArgs& A, const double2* buf, int64_t g0, int nf) {
  const int F = A.F, m = A.m;
  for (int idx = threadIdx.x; idx < F * m; idx += blockDim.x) {
    int f, k;
    split<STRIDED>(idx, F, m, f, k);
    if (f >= nf) continue;
    const Geo q = geo<STRIDED>(A, g0 + f);
    const double2 z = buf[f * A.fs + k];
    if (STRIDED) *reinterpret_cast<double2*>(A.out + q.bx + k * q.st) = z;
    else {
      A.out[q.bx + k] = z.x;
      if (q.by >= 0) A.out[q.by + k] = z.y;
    }
  }
}

template <bool STRIDED, bool EPI>
__device__ void store_packed(const PassArgs& A, const double2* buf, int64_t g0, int nf, double& acc) {
  const int F = A.F, h = A.h, m = A.m;
  for (int idx = threadIdx.x; idx < F * h; idx += blockDim.x) {
    int f, j;
    split<STRIDED>(idx, F, h, f, j);
    if (f >= nf) continue;
    const Geo q = geo<STRIDED>(A, g0 + f);
    const double2* fib = buf + f * A.fs;
    double xa, xb, ya, yb;  // x/y packed values at rows (j ? j+1 : 0) and (j ? j+h : 1)
    if (j == 0) {
      const double2 z0 = fib[0], zh = fib[h];
      xa = A.c0 * z0.x; ya = A.c0 * z0.y;
      xb = A.c0 * zh.x; yb = A.c0 * zh.y;
    } else {
      const double2 a = fib[j], b = fib[m - j];
      xa = A.c1 * (a.x + b.x);
      xb = A.c1 * (a.y - b.y);
      ya = A.c1 * (a.y + b.y);
      yb = A.c1 * (b.x - a.x);
    }
    const int64_t ia = q.st * (j ? j + 1 : 0), ib = q.st * (j ? j + h : 1);
    if (STRIDED && !EPI) {
      *reinterpret_cast<double2*>(A.out + q.bx + ia) = make_double2(xa, ya);
      *reinterpret_cast<double2*>(A.out + q.bx + ib) = make_double2(xb, yb);
    } else {
      put<STRIDED, EPI>(A, q.bx + ia, xa, acc);
      put<STRIDED, EPI>(A, q.bx + ib, xb, acc);
      if (q.by >= 0) {
        put<STRIDED, EPI>(A, q.by + ia, ya, acc);
        put<STRIDED, EPI>(A, q.by + ib, yb, acc);
      }
    }
  }
}

template <bool STRIDED, int KIND, bool EPI>
__global__ void __launch_bounds__(kThreads) axis_pass(const PassArgs A) {
  extern __shared__ double2 smem[];
  __shared__ double red[32];
  double2* b0 = smem;
  double2* b1 = smem + A.F * A.fs;
  double acc = 0.0, nrm = 0.0;
  for (int64_t tile = blockIdx.x; tile * A.F < A.G; tile += gridDim.x) {
    const int64_t g0 = tile * A.F;
    const int64_t rem = A.G - g0;
    const int nf = rem < A.F ? (int)rem : A.F;
    double2* res;
    if (KIND == K_ANALYZE) {
      load_plain<STRIDED>(A, b0, g0, nf);
      __syncthreads();
      res = fft_tile(b0, b1, A.F, A.fs, A.plan, -1);
    } else {
      load_packed<STRIDED>(A, b0, g0, nf);
      __syncthreads();
      res = fft_tile(b0, b1, A.F, A.fs, A.plan, +1);
      if (KIND == K_GRAM || KIND == K_RESID) {
        apply_mask<KIND == K_RESID>(A, res, g0, nf, nrm);
        __syncthreads();
        res = fft_tile(res, res == b0 ? b1 : b0, A.F, A.fs, A.plan, -1);
      }
    }
    if (KIND == K_SYNTH) store_plain<STRIDED>(A, res, g0, nf);
    else store_packed<STRIDED, EPI>(A, res, g0, nf, acc);
    __syncthreads();
  }
  if (EPI && A.epi.partials) {
    const double s = block_reduce(acc, SumOp(), red);
    if (threadIdx.x == 0) A.epi.partials[blockIdx.x] = s;
  }
  if (KIND == K_GRAM && A.nrm_partials) {
    const double s = block_reduce(nrm, SumOp(), red);
    if (threadIdx.x == 0) A.nrm_partials[blockIdx.x] = s;
  }
}

template <bool S>
KernelFn pick_kernel(int kind, bool epi) {
  switch (kind) {
    case K_SYNTH: return axis_pass<S, K_SYNTH, false>;
    case K_ANALYZE: return epi ? axis_pass<S, K_ANALYZE, true> : axis_pass<S, K_ANALYZE, false>;
    case K_GRAM: return epi ? axis_pass<S, K_GRAM, true> : axis_pass<S, K_GRAM, false>;
    default: return epi ? axis_pass<S, K_RESID, true> : axis_pass<S, K_RESID, false>;
  }
}

int set_smem_attr(KernelFn k) {
  static_assert(kSmemBudget <= 227 * 1024, "smem budget");
  cudaFuncAttributes fa;
  FL_CUDA(cudaFuncGetAttributes(&fa, k));
  const int limit = 227 * 1024 - (int)fa.sharedSizeBytes;
  FL_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, limit));
  return FL_OK;
}

}  // namespace

int run_pass(const fl_plan* p, int axis, int kind, const double* in, double* out,
             const uint32_t* bits, const double* bhat, const KktEpi* epi, int* nblocks,
             cudaStream_t s) {
  return run_pass_n(p, axis, kind, in, out, bits, bhat, epi, nblocks, nullptr, s);
}

int run_pass_n(const fl_plan* p, int axis, int kind, const double* in, double* out,
               const uint32_t* bits, const double* bhat, const KktEpi* epi, int* nblocks,
               double* nrm_partials, cudaStream_t s) {
  static std::mutex attrs_mu;
  static bool attrs_set[kMaxDevices][2][4][2] = {};  // per-device smem opt-in
  const bool strided = axis < p->ndim - 1;
  if (!p->planned[axis]) return fail(FL_E_VALUE, "axis " + std::to_string(axis) + " is a batch extent of this plan");
  if ((kind == K_GRAM || kind == K_RESID) && strided) {
    // only the strided fused gram of the axis-0-last order (kkt_order_b)
    int64_t in_ = 1;
    for (int a = axis + 1; a < p->ndim; ++a) in_ *= p->dims[a];
    if (kind != K_GRAM || p->dims[axis] != 512 || in_ % 32 != 0 || nrm_partials)
      return fail(FL_E_VALUE, "a strided fused mask pass needs the gram kind, m = 512, rows of 32k voxels "
                              "and no norm partials");
  }
  PassArgs A;
  A.in = in;
  A.out = out;
  A.m = (int)p->dims[axis];
  A.h = A.m / 2;
  int64_t outer = 1, inner = 1;
  for (int a = 0; a < axis; ++a) outer *= p->dims[a];
  for (int a = axis + 1; a < p->ndim; ++a) inner *= p->dims[a];
  if (strided) {
    A.inner = inner;
    A.G = outer * (inner / 2);
    A.has_y = 1;
  } else {
    A.inner = 1;
    A.has_y = outer >= 2;
    A.G = A.has_y ? outer / 2 : 1;
  }
  A.c0 = 1.0 / std::sqrt((double)A.m);
  A.c1 = 1.0 / std::sqrt(2.0 * (double)A.m);
  A.plan = p->axis[axis];
  A.bits = bits;
  A.bhat = bhat;
  A.nrm_partials = nrm_partials;
  if (epi) A.epi = *epi;
  if (p->lng[axis].on) return run_long(p, axis, kind, A, strided, epi, nblocks, s);
  if (fast_supported(A.m)) return launch_fast(A.m, strided, kind, epi != nullptr, A, nblocks, s);
  A.fs = A.m + 1;
  const int per_fibre = 2 * A.fs * (int)sizeof(double2);
  if (per_fibre > 226 * 1024)
    return fail(FL_E_SHAPE, "axis length " + std::to_string(A.m) + " exceeds the shared-memory FFT limit");
  int F = std::max(1, std::min(16, kSmemBudget / per_fibre));
  if (F >= 8) F = F / 8 * 8;
  if ((int64_t)F > A.G) F = (int)A.G;
  A.F = F;
  const bool has_epi = epi != nullptr;
  KernelFn k = strided ? pick_kernel<true>(kind, has_epi) : pick_kernel<false>(kind, has_epi);
  int dev = 0;
  FL_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(FL_E_VALUE, "device index out of range");
  {
    std::lock_guard<std::mutex> lock(attrs_mu);
    bool& done = attrs_set[dev][strided][kind][has_epi];
    if (!done) {
      FL_TRY(set_smem_attr(k));
      done = true;
    }
  }
  const int64_t tiles = (A.G + F - 1) / F;
  const int grid = (int)std::min<int64_t>(tiles, kMaxGrid);
  const size_t smem = (size_t)per_fibre * F;
  k<<<grid, kThreads, smem, s>>>(A);
  FL_LAUNCH_CHECK();
  if (nblocks) *nblocks = grid;
  return FL_OK;
}

int op_synthesize(const fl_plan* p, const double* in, double* out, cudaStream_t s) {
  const double* src = in;
  for (int a = 0; a < p->ndim; ++a) {
    FL_TRY(run_pass(p, a, K_SYNTH, src, out, nullptr, nullptr, nullptr, nullptr, s));
    src = out;
  }
  return FL_OK;
}

int op_analyze(const fl_plan* p, const double* in, double* out, cudaStream_t s) {
  const double* src = in;
  for (int a = p->ndim - 1; a >= 0; --a) {
    FL_TRY(run_pass(p, a, K_ANALYZE, src, out, nullptr, nullptr, nullptr, nullptr, s));
    src = out;
  }
  return FL_OK;
}

// KKT apply operator order.  Default (order A): synthesis along axes
// 0..d-2, the fused mask pass on the contiguous axis, analysis back along
// d-2..0, then the KKT epilogue as a separate 16-byte elementwise pass (fused
// into the last, strided, analysis its four operand streams load in 128-byte
// row segments after the tile's FFT: 44 % of HBM, round 1).
// Order B (3D, axis 0 and the contiguous axis of length 512): synthesis along
// the contiguous axis first, the fused mask pass on axis 0 (strided, mirrored
// engine), analysis ending on the contiguous axis with the epilogue fused in
// (group pass; its operand rows are prefetched into L2 when the pair starts):
// 120.125 instead of 136.125 executed B/voxel.  Measured at 512^3: 3.46 ->
// 3.24 ms per matvec (the strided fused gram costs 0.80 ms against 0.65 ms on
// the contiguous axis, the fused analysis + epilogue 1.25 ms against 0.39 +
// 1.12 ms).  At 1024^3 the strided fused gram (7.9 ms against 4.7) and the
// fused 1024-point analysis (15 ms) lose, so order A stays there.
bool kkt_order_b(const fl_plan* p) {
  return p->ndim == 3 && p->dims[0] == 512 && p->dims[2] == 512 && !p->lng[0].on && !p->lng[2].on &&
         (p->dims[1] * p->dims[2]) % 32 == 0;
}

int op_gram(const fl_plan* p, const uint32_t* bits, const double* bhat, bool resid,
            const double* in, double* out, const KktEpi* epi, int* nblocks, cudaStream_t s) {
  if (epi && !resid && kkt_order_b(p)) {
    const int d = p->ndim;
    const double* src = in;
    for (int a = d - 1; a >= 1; --a) {
      FL_TRY(run_pass(p, a, K_SYNTH, src, out, nullptr, nullptr, nullptr, nullptr, s));
      src = out;
    }
    FL_TRY(run_pass(p, 0, K_GRAM, src, out, bits, nullptr, nullptr, nullptr, s));
    for (int a = 1; a < d; ++a)
      FL_TRY(run_pass(p, a, K_ANALYZE, out, out, nullptr, nullptr, a == d - 1 ? epi : nullptr,
                      a == d - 1 ? nblocks : nullptr, s));
    return FL_OK;
  }
  if (epi && p->ndim > 1) {
    FL_TRY(op_gram(p, bits, bhat, resid, in, out, nullptr, nullptr, s));
    return kkt_epilogue(p->n, out, epi->pb, epi->pz, epi->sig1, epi->sig2, epi->bottom, epi->partials,
                        nblocks, s);
  }
  const int d = p->ndim;
  const int mid = resid ? K_RESID : K_GRAM;
  if (d == 1) return run_pass(p, 0, mid, in, out, bits, bhat, epi, nblocks, s);
  const double* src = in;
  for (int a = 0; a < d - 1; ++a) {
    FL_TRY(run_pass(p, a, K_SYNTH, src, out, nullptr, nullptr, nullptr, nullptr, s));
    src = out;
  }
  FL_TRY(run_pass(p, d - 1, mid, src, out, bits, bhat, nullptr, nullptr, s));
  for (int a = d - 2; a >= 0; --a)
    FL_TRY(run_pass(p, a, K_ANALYZE, out, out, nullptr, nullptr, a == 0 ? epi : nullptr,
                    a == 0 ? nblocks : nullptr, s));
  return FL_OK;
}

// g = G beta with the fused-pass partials of ||Z A beta||^2 = beta . G beta
// (the matrix part of the PCG curvature).  Returns FL_E_VALUE via *have_norm
// = false when the mask pass cannot produce them (four-step long axis).
int op_gram_norm(const fl_plan* p, const uint32_t* bits, const double* in, double* out,
                 double* nrm_partials, int* nblocks, bool* have_norm, cudaStream_t s) {
  const int d = p->ndim;
  *have_norm = !p->lng[d - 1].on;
  double* np = *have_norm ? nrm_partials : nullptr;
  if (d == 1) return run_pass_n(p, 0, K_GRAM, in, out, bits, nullptr, nullptr, nblocks, np, s);
  const double* src = in;
  for (int a = 0; a < d - 1; ++a) {
    FL_TRY(run_pass(p, a, K_SYNTH, src, out, nullptr, nullptr, nullptr, nullptr, s));
    src = out;
  }
  FL_TRY(run_pass_n(p, d - 1, K_GRAM, src, out, bits, nullptr, nullptr, nblocks, np, s));
  for (int a = d - 2; a >= 0; --a)
    FL_TRY(run_pass(p, a, K_ANALYZE, out, out, nullptr, nullptr, nullptr, nullptr, s));
  return FL_OK;
}

}  // namespace fl
