// Axis passes for fibres longer than one CTA's shared memory (m > 8192,
// non-power-of-two m > 6144): four-step FFT through a plan-owned complex
// scratch vector.  Used for the reference's long 1D cases (test_fourier
// 2^20, test_ipm 2^14); never on the 3D hot path.
//
// For a fibre pair c[t] = x[t] + i y[t] (synthesis: the unpacked combined
// spectrum), with m = m1 * m2 and t = t1*m2 + t2:
//   A  length-m1 FFTs over t1 (stride m2) for every t2, then the twiddle
//      exp(sign 2 pi i t2 k1 / m)                       (k_four_a)
//   C  length-m2 FFTs over t2 (contiguous) for every k1  (k_four_c)
// leaves X[k1 + m1 k2] at index k1*m2 + k2 (transposed order), which the
// store stage reads through pos(k) = (k % m1) * m2 + k / m1.
#include <algorithm>
#include <cmath>
#include <string>

#include "fl_common.cuh"
#include "fl_internal.h"
#include "fl_passargs.cuh"

namespace fl {
namespace {

constexpr int T = 256;
constexpr int kSubBudget = 196 * 1024;

struct LongArgs {
  PassArgs A;
  double2* c;  // scratch, G * m complex
  int m1, m2;
  AxisPlan p1, p2;
};

__device__ __forceinline__ int64_t pos(int64_t k, int m1, int m2) { return (k % m1) * m2 + k / m1; }

template <bool STRIDED, bool SYNTH>
__global__ void k_four_load(const LongArgs L) {
  const PassArgs& A = L.A;
  const int m = A.m, h = A.h;
  const int64_t per = SYNTH ? h : m;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A.G * per;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = i / per;
    const int j = (int)(i - g * per);
    const Geo Q = geo<STRIDED>(A, g);
    double2* cf = L.c + g * m;
    if (!SYNTH) {
      double2 z = make_double2(A.in[Q.bx + j * Q.st], 0.0);
      if (Q.by >= 0) z.y = A.in[Q.by + j * Q.st];
      cf[j] = z;
      continue;
    }
    const int64_t ia = Q.st * (j ? j + 1 : 0), ib = Q.st * (j ? j + h : 1);
    const double xa = A.in[Q.bx + ia], xb = A.in[Q.bx + ib];
    const double ya = Q.by >= 0 ? A.in[Q.by + ia] : 0.0, yb = Q.by >= 0 ? A.in[Q.by + ib] : 0.0;
    if (j == 0) {
      cf[0] = make_double2(A.c0 * xa, A.c0 * ya);
      cf[h] = make_double2(A.c0 * xb, A.c0 * yb);
    } else {
      cf[j] = make_double2(A.c1 * (xa - yb), A.c1 * (xb + ya));
      cf[m - j] = make_double2(A.c1 * (xa + yb), A.c1 * (ya - xb));
    }
  }
}

// Batched complex FFT of F fibres per tile from the scratch vector.
// A_STEP: fibres (g, t2), length m1, stride m2, twiddled on store.
// otherwise: fibres (g, k1), length m2, contiguous.
template <bool A_STEP>
__global__ void k_four_fft(const LongArgs L, int sign, int F, int fs) {
  extern __shared__ double2 sm[];
  const int m = L.A.m, m1 = L.m1, m2 = L.m2;
  const int len = A_STEP ? m1 : m2;
  const int per = A_STEP ? m2 : m1;  // fibres per pair
  const AxisPlan& P = A_STEP ? L.p1 : L.p2;
  const int64_t nfib = L.A.G * per;
  double2* b0 = sm;
  double2* b1 = sm + F * fs;
  for (int64_t f0 = (int64_t)blockIdx.x * F; f0 < nfib; f0 += (int64_t)gridDim.x * F) {
    for (int idx = threadIdx.x; idx < F * len; idx += blockDim.x) {
      const int f = idx % F, k = idx / F;
      const int64_t fi = f0 + f;
      double2 z = make_double2(0.0, 0.0);
      if (fi < nfib) {
        const int64_t g = fi / per, r = fi - g * per;
        z = A_STEP ? L.c[g * m + (int64_t)k * m2 + r] : L.c[g * m + r * m2 + k];
      }
      b0[f * fs + k] = z;
    }
    __syncthreads();
    double2* res = fft_tile(b0, b1, F, fs, P, sign);
    for (int idx = threadIdx.x; idx < F * len; idx += blockDim.x) {
      const int f = idx % F, k = idx / F;
      const int64_t fi = f0 + f;
      if (fi >= nfib) continue;
      const int64_t g = fi / per, r = fi - g * per;
      double2 z = res[f * fs + k];
      if (A_STEP) {
        // exp(sign 2 pi i r k / m) with r = t2, k = k1
        const int64_t e = (r * (int64_t)k) % m;
        double s, co;
        sincospi(2.0 * (double)e / (double)m, &s, &co);
        z = cmul(z, make_double2(co, sign * s));
        L.c[g * m + (int64_t)k * m2 + r] = z;
      } else {
        L.c[g * m + r * m2 + k] = z;
      }
    }
    __syncthreads();
  }
}

template <bool STRIDED, bool SYNTH, bool EPI>
__global__ void k_four_store(const LongArgs L) {
  __shared__ double red[32];
  const PassArgs& A = L.A;
  const int m = A.m, h = A.h, m1 = L.m1, m2 = L.m2;
  const int64_t per = SYNTH ? m : h;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A.G * per;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = i / per;
    const int j = (int)(i - g * per);
    const Geo Q = geo<STRIDED>(A, g);
    const double2* cf = L.c + g * m;
    if (SYNTH) {
      const double2 z = cf[pos(j, m1, m2)];
      A.out[Q.bx + j * Q.st] = z.x;
      if (Q.by >= 0) A.out[Q.by + j * Q.st] = z.y;
      continue;
    }
    double xa, xb, ya, yb;
    if (j == 0) {
      const double2 z0 = cf[pos(0, m1, m2)], zh = cf[pos(h, m1, m2)];
      xa = A.c0 * z0.x; ya = A.c0 * z0.y;
      xb = A.c0 * zh.x; yb = A.c0 * zh.y;
    } else {
      const double2 a = cf[pos(j, m1, m2)], b = cf[pos(m - j, m1, m2)];
      xa = A.c1 * (a.x + b.x);
      xb = A.c1 * (a.y - b.y);
      ya = A.c1 * (a.y + b.y);
      yb = A.c1 * (b.x - a.x);
    }
    const int64_t ia = Q.st * (j ? j + 1 : 0), ib = Q.st * (j ? j + h : 1);
    put<STRIDED, EPI>(A, Q.bx + ia, xa, acc);
    put<STRIDED, EPI>(A, Q.bx + ib, xb, acc);
    if (Q.by >= 0) {
      put<STRIDED, EPI>(A, Q.by + ia, ya, acc);
      put<STRIDED, EPI>(A, Q.by + ib, yb, acc);
    }
  }
  if (EPI && A.epi.partials) {
    const double s = block_reduce(acc, SumOp(), red);
    if (threadIdx.x == 0) A.epi.partials[blockIdx.x] = s;
  }
}

template <bool RESID>
__global__ void k_mask_full(int64_t n, const uint32_t* __restrict__ bits, const double* __restrict__ bhat,
                            double* __restrict__ x) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const bool miss = missing(bits, v);
    x[v] = miss ? 0.0 : (RESID ? bhat[v] - x[v] : x[v]);
  }
}

int sub_tiles(int len, int* F, int* fs, size_t* smem) {
  *fs = len + 1;
  const int per = 2 * (*fs) * 16;
  if (per > kSubBudget) return fail(FL_E_SHAPE, "four-step factor too long for shared memory");
  *F = std::max(1, std::min(16, kSubBudget / per));
  *smem = (size_t)per * (*F);
  return FL_OK;
}

template <class K>
int allow_smem(K k) {
  cudaFuncAttributes fa;
  FL_CUDA(cudaFuncGetAttributes(&fa, k));
  FL_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               227 * 1024 - (int)fa.sharedSizeBytes));
  return FL_OK;
}

int four_step_fft(const LongArgs& L, int sign, cudaStream_t s) {
  int F, fs;
  size_t smem;
  FL_TRY(sub_tiles(L.m1, &F, &fs, &smem));
  FL_TRY(allow_smem(k_four_fft<true>));
  int64_t nf = L.A.G * L.m2;
  int grid = (int)std::min<int64_t>((nf + F - 1) / F, 148 * 8);
  k_four_fft<true><<<grid, T, smem, s>>>(L, sign, F, fs);
  FL_LAUNCH_CHECK();
  FL_TRY(sub_tiles(L.m2, &F, &fs, &smem));
  FL_TRY(allow_smem(k_four_fft<false>));
  nf = L.A.G * L.m1;
  grid = (int)std::min<int64_t>((nf + F - 1) / F, 148 * 8);
  k_four_fft<false><<<grid, T, smem, s>>>(L, sign, F, fs);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int grid_n(int64_t n) { return (int)std::min<int64_t>((n + T - 1) / T, 148 * 16); }

template <bool S>
int four_pass(const LongArgs& L, bool synth, const KktEpi* epi, int* nblocks, cudaStream_t s) {
  const int64_t work_load = L.A.G * (synth ? L.A.h : L.A.m);
  if (synth) k_four_load<S, true><<<grid_n(work_load), T, 0, s>>>(L);
  else k_four_load<S, false><<<grid_n(work_load), T, 0, s>>>(L);
  FL_LAUNCH_CHECK();
  FL_TRY(four_step_fft(L, synth ? +1 : -1, s));
  const int64_t work_store = L.A.G * (synth ? L.A.m : L.A.h);
  const int grid = grid_n(work_store);
  if (synth) k_four_store<S, true, false><<<grid, T, 0, s>>>(L);
  else if (epi) k_four_store<S, false, true><<<grid, T, 0, s>>>(L);
  else k_four_store<S, false, false><<<grid, T, 0, s>>>(L);
  FL_LAUNCH_CHECK();
  if (nblocks) *nblocks = grid;
  return FL_OK;
}

}  // namespace

int long_factor(int m, int* m1, int* m2) {
  // balanced m = m1 * m2 with both factors fitting the shared-memory engine
  const int cap = (kSubBudget / 32) - 1;
  int best = 0;
  for (int a = 2; (int64_t)a * a <= m; ++a)
    if (m % a == 0 && a <= cap && m / a <= cap) best = a;
  if (!best) return fail(FL_E_SHAPE, "axis length " + std::to_string(m) +
                                         " has no factorisation into two shared-memory FFTs");
  *m1 = best;
  *m2 = m / best;
  return FL_OK;
}

int run_long(const fl_plan* p, int axis, int kind, const PassArgs& A0, bool strided,
             const KktEpi* epi, int* nblocks, cudaStream_t s) {
  const LongAxis& la = p->lng[axis];
  LongArgs L;
  L.A = A0;
  L.c = la.scratch;
  L.m1 = la.m1;
  L.m2 = la.m2;
  L.p1 = la.p1;
  L.p2 = la.p2;
  if (kind == K_SYNTH || kind == K_ANALYZE) {
    return strided ? four_pass<true>(L, kind == K_SYNTH, epi, nblocks, s)
                   : four_pass<false>(L, kind == K_SYNTH, epi, nblocks, s);
  }
  // fused mask pass on a long last axis: synthesize, mask on the grid, analyze
  L.A.epi = KktEpi();
  FL_TRY(strided ? four_pass<true>(L, true, nullptr, nullptr, s) : four_pass<false>(L, true, nullptr, nullptr, s));
  if (kind == K_RESID) k_mask_full<true><<<grid_n(p->n), T, 0, s>>>(p->n, A0.bits, A0.bhat, A0.out);
  else k_mask_full<false><<<grid_n(p->n), T, 0, s>>>(p->n, A0.bits, A0.bhat, A0.out);
  FL_LAUNCH_CHECK();
  L.A = A0;
  L.A.in = A0.out;
  return strided ? four_pass<true>(L, false, epi, nblocks, s) : four_pass<false>(L, false, epi, nblocks, s);
}

}  // namespace fl
