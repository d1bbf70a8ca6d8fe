// Group-decoupled contiguous-axis passes (fibre lengths 512, 1024, 2048).
//
// The CTA-tiled engine (fast_pass) runs W fibre pairs per CTA in lock step:
// every shared-memory exchange of every fibre is a CTA-wide barrier, and the
// next tile's staging waits for all of them -- at 512^3 the fused gram pass
// spent its time in barrier / short-scoreboard stalls with few warps able to
// issue (round-1 ncu: 44 % of HBM peak, 23 % warps active).
//
// Here a fibre pair is owned by ONE GROUP of P = M/E threads (two warps at
// m = 512 and 1024) that walks its own sequence of pairs (pair g, g + NG x
// gridDim, ...) with its own:
//   * TMA row stage (cp.async.bulk of the pair's two contiguous rows into a
//     planar stage, completing on the group's mbarrier, issued by the group
//     leader),
//   * exchange buffers (two, alternating: one named barrier per exchange
//     instead of two),
//   * named barrier (bar.sync 1 + group, P).
// No barrier spans groups inside the loop, so the NG groups of a CTA (and the
// groups of every resident CTA) drift independently and hide each other's
// exchange and load latency.  The stage is refilled as soon as the group has
// passed the first exchange of the FFT that follows its last read (the
// residual pass streams its b_hat rows through the same stage between the
// two FFTs), so no extra shared memory is needed for prefetching.
//
// The FFT itself (radix stages, twiddles, natural layout, pack/unpack with
// the reference's scaling fourier.py:172-198) is the fast:: engine; the mask
// of the fused pass (masking.py:107-118) is applied in registers, its bits
// gathered once per pair by warp shuffles from one word per lane.
#pragma once

#include "fl_fastpass.cuh"

namespace fl {
namespace gpk {

using fast::Geom;
using fast::si;

__device__ __forceinline__ void group_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// CFG of the fast:: geometry used for the FFT (E = 8 up to 512, 16 above)
template <int M>
struct GCfg {
  static constexpr int CFG = fast::cfg_code(0, 0, 2);
  using G = Geom<M, CFG>;
  static constexpr int E = G::E, P = G::P, FS = G::FS;
  static constexpr int NG = M <= 1024 ? 4 : 2;  // groups per CTA
  static constexpr int T = NG * P;
  static constexpr int GD2 = 2 * FS + M;           // double2 per group: 2 exchange buffers + row stage
  static constexpr int SMEM = NG * GD2 * 16;
  static constexpr int MINB = M <= 512 ? 2 : 1;    // CTAs per SM asked of __launch_bounds__
};

// FFT with one named barrier per exchange (alternating buffers); ``hook`` runs
// once, right after the first barrier (every thread of the group has passed
// all its earlier shared-memory reads by then).
template <int M, int CFG, int S = 0, class F>
__device__ __forceinline__ void gfft(double2* v, double2* fA, double2* fB, int& buf, int q, const double2* tw,
                                     int sign, int bid, F&& hook) {
  using G = Geom<M, CFG>;
  fast::stage_compute<M, CFG, S>(v, q, tw, sign);
  if constexpr (S + 1 < G::NST) {
    double2* f = buf ? fB : fA;
    fast::stage_store<M, CFG, S>(v, f, q);
    group_sync(bid, G::P);
    if constexpr (S == 0) hook();
    fast::load_natural<M, CFG>(v, f, q);
    buf ^= 1;
    gfft<M, CFG, S + 1>(v, fA, fB, buf, q, tw, sign, bid, hook);
  } else if constexpr (S == 0) {
    hook();
  }
}

// Leader: TMA the pair's rows (x, and y when present) into the planar stage.
template <int M>
__device__ __forceinline__ void tma_rows(const double* src, const Geo& Q, double* stage, unsigned long long* bar) {
  fence_proxy_async();  // order the group's generic reads of the stage before the async writes
  fast::mbar_expect_tx(bar, (Q.by >= 0 ? 2u : 1u) * M * 8u);
  fast::bulk_g2s(stage, src + Q.bx, M * 8u, bar);
  if (Q.by >= 0) fast::bulk_g2s(stage + M, src + Q.by, M * 8u, bar);
}

template <int M, int KIND, bool EPI>
__global__ void __launch_bounds__(GCfg<M>::T, GCfg<M>::MINB) group_pass(const PassArgs A) {
  using C = GCfg<M>;
  constexpr int CFG = C::CFG, E = C::E, P = C::P, NG = C::NG, H = M / 2, FS = C::FS;
  constexpr bool SHFL_PACK = P == 64 && E == 8;
  constexpr bool MASKED = KIND == K_GRAM || KIND == K_RESID;
  extern __shared__ double2 smem[];
  __shared__ double red[32];
  __shared__ unsigned long long gbar[NG][2];
  const int c = threadIdx.x / P, tg = threadIdx.x % P;
  int q = tg, partner = 0;
  if constexpr (SHFL_PACK) {
    int cc;
    fpk::lane_map_pair64(tg, cc, q, partner);
  }
  double2* fA = smem + c * C::GD2;
  double2* fB = fA + FS;
  double* stage = reinterpret_cast<double*>(fA + 2 * FS);
  unsigned long long* bar = gbar[c];
  const int bid = 1 + c;
  const bool leader = tg == 0;
  const double2* tw = A.plan.tw;
  const double c0 = A.c0, c1 = A.c1;
  // pair indices fit 32 bits (the launcher falls back to the CTA-tiled engine otherwise)
  const int gstride = (int)gridDim.x * NG;
  const int npairs = (int)A.G;
  int g = (int)blockIdx.x * NG + c;
  if (leader) {
    fast::mbar_init(bar, 1);
    fast::mbar_init(bar + 1, 1);
  }
  __syncthreads();
  if (leader && g < npairs) tma_rows<M>(A.in, geo<false>(A, g), stage, bar);
  unsigned ph0 = 0, ph1 = 0;
  int buf = 0;
  double acc = 0.0, nrm = 0.0;
  for (; g < npairs; g += gstride) {
    const Geo Q = geo<false>(A, g);
    const int gn = g + gstride;
    const bool has_y = Q.by >= 0;
    // refill of the stage with the next pair's rows (after the stage's last read)
    auto refill_next = [&]() {
      if (leader && gn < npairs) tma_rows<M>(A.in, geo<false>(A, gn), stage, bar);
    };
    if constexpr (EPI) {
      // the KKT epilogue's operand rows of this pair (read after the FFT): into L2 now
      if (leader) {
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          const double* src = o == 0 ? A.epi.pb : o == 1 ? A.epi.pz : o == 2 ? A.epi.sig1 : A.epi.sig2;
          fast::bulk_prefetch_l2(src + Q.bx, M * 8u);
          if (has_y) fast::bulk_prefetch_l2(src + Q.by, M * 8u);
        }
      }
    }
    fast::mbar_wait(bar, ph0);
    ph0 ^= 1u;
    double2 v[E];
    if constexpr (KIND == K_ANALYZE) {
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const int k = q + r * P;
        v[r] = make_double2(stage[k], has_y ? stage[M + k] : 0.0);
      }
    } else {
      // unpack (fourier.py:176-181 with the ortho scale) straight from the
      // staged rows: Zin_k needs rows (k+1, k+H) for k < H, (M-k+1, M-k+H) above
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const int k = q + r * P;
        const bool lo = r < E / 2;
        const int j = lo ? k : M - k;
        const bool edge = q == 0 && (r == 0 || r == E / 2);
        const int ia = edge ? (r == 0 ? 0 : 1) : j + 1;
        const double ax = stage[ia], ay = has_y ? stage[M + ia] : 0.0;
        if (edge) {
          v[r] = make_double2(c0 * ax, c0 * ay);
        } else {
          const double bx = stage[j + H], by = has_y ? stage[M + j + H] : 0.0;
          v[r] = lo ? make_double2(c1 * (ax - by), c1 * (bx + ay)) : make_double2(c1 * (ax + by), c1 * (ay - bx));
        }
      }
    }
    uint32_t mbits = 0;
    if constexpr (MASKED) {
      // one mask word per lane (row x words, then row y words), bits gathered by shuffle
      constexpr int WPR = M / 32;  // words per row
      const int lane = threadIdx.x & 31;
      if constexpr (WPR <= 16) {
        uint32_t word = 0;
        if (lane < WPR) word = __ldg(A.bits + (Q.bx >> 5) + lane);
        else if (lane >= 16 && lane < 16 + WPR && has_y) word = __ldg(A.bits + (Q.by >> 5) + lane - 16);
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int t = q + r * P;
          const uint32_t wx = __shfl_sync(0xffffffffu, word, t >> 5);
          const uint32_t wy = __shfl_sync(0xffffffffu, word, 16 + (t >> 5));
          mbits |= ((wx >> (t & 31)) & 1u) << (2 * r);
          mbits |= ((wy >> (t & 31)) & 1u) << (2 * r + 1);
        }
      } else {
        static_assert(WPR % 32 == 0, "mask rows of whole warps");
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int t = q + r * P;
          const int wi = t >> 5;  // word of this sample: one per lane in each 32-word chunk
          const uint32_t wxl = __ldg(A.bits + (Q.bx >> 5) + (wi & ~31) + lane);
          const uint32_t wyl = has_y ? __ldg(A.bits + (Q.by >> 5) + (wi & ~31) + lane) : 0u;
          const uint32_t wx = __shfl_sync(0xffffffffu, wxl, wi & 31);
          const uint32_t wy = __shfl_sync(0xffffffffu, wyl, wi & 31);
          mbits |= ((wx >> (t & 31)) & 1u) << (2 * r);
          mbits |= ((wy >> (t & 31)) & 1u) << (2 * r + 1);
        }
      }
    }
    if constexpr (KIND == K_ANALYZE) {
      gfft<M, CFG>(v, fA, fB, buf, q, tw, -1, bid, refill_next);
    } else {
      if constexpr (KIND == K_RESID) {
        // the stage is free after the first exchange: stream this pair's b_hat rows in
        gfft<M, CFG>(v, fA, fB, buf, q, tw, +1, bid, [&]() {
          if (leader) tma_rows<M>(A.bhat, Q, stage, bar + 1);
        });
      } else {
        gfft<M, CFG>(v, fA, fB, buf, q, tw, +1, bid, refill_next);
      }
      if constexpr (KIND == K_SYNTH) {
        double* px = A.out + Q.bx + q;
        double* py = A.out + Q.by + q;
#pragma unroll
        for (int r = 0; r < E; ++r) {
          px[r * P] = v[r].x;
          if (has_y) py[r * P] = v[r].y;
        }
      } else {
        if constexpr (KIND == K_RESID) {
          fast::mbar_wait(bar + 1, ph1);
          ph1 ^= 1u;
        }
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int t = q + r * P;
          double2 z = v[r];
          const bool mx = (mbits >> (2 * r)) & 1u, my = (mbits >> (2 * r + 1)) & 1u;
          if (KIND == K_RESID) {
            z.x = mx ? 0.0 : stage[t] - z.x;
            z.y = (!has_y || my) ? 0.0 : stage[M + t] - z.y;
          } else {
            if (mx) z.x = 0.0;
            if (!has_y || my) z.y = 0.0;
            nrm += z.x * z.x + z.y * z.y;  // ||Z A beta||^2 = beta . G beta
          }
          v[r] = z;
        }
        if constexpr (KIND == K_RESID) gfft<M, CFG>(v, fA, fB, buf, q, tw, -1, bid, refill_next);
        else gfft<M, CFG>(v, fA, fB, buf, q, tw, -1, bid, []() {});
      }
    }
    if constexpr (KIND != K_SYNTH) {
      // pack (fourier.py:193-197): rows (j+1, j+H) from Z_j and Z_{M-j}
      if constexpr (SHFL_PACK) {
        double2 mir[E / 2];
#pragma unroll
        for (int r = 0; r < E / 2; ++r) {
          const double2 sh = fpk::shfl2(v[E - 1 - r], partner);
          mir[r] = q == 0 ? v[(E - r) & (E - 1)] : sh;
        }
#pragma unroll
        for (int r = 0; r < E / 2; ++r) {
          const int j = q + r * P;
          const bool j0 = r == 0 && q == 0;
          const double2 a = v[r], b = mir[r];
          double xa, xb, ya, yb;
          if (j0) {
            const double2 zh = v[E / 2];
            xa = c0 * a.x; ya = c0 * a.y;
            xb = c0 * zh.x; yb = c0 * zh.y;
          } else {
            xa = c1 * (a.x + b.x);
            xb = c1 * (a.y - b.y);
            ya = c1 * (a.y + b.y);
            yb = c1 * (b.x - a.x);
          }
          const int64_t ia = j0 ? 0 : j + 1, ib = j0 ? 1 : j + H;
          put<false, EPI>(A, Q.bx + ia, xa, acc);
          put<false, EPI>(A, Q.bx + ib, xb, acc);
          if (has_y) {
            put<false, EPI>(A, Q.by + ia, ya, acc);
            put<false, EPI>(A, Q.by + ib, yb, acc);
          }
        }
      } else {
        double2* f = buf ? fB : fA;
        fast::store_natural<M, CFG>(v, f, q);
        group_sync(bid, P);
        buf ^= 1;
        const int qm = -q + ((-q) >> 3);
#pragma unroll
        for (int r = 0; r < E / 2; ++r) {
          const int j = q + r * P;
          const bool j0 = r == 0 && q == 0;
          double xa, xb, ya, yb;
          if (j0) {
            const double2 z0 = f[0], zh = f[si(H)];
            xa = c0 * z0.x; ya = c0 * z0.y;
            xb = c0 * zh.x; yb = c0 * zh.y;
          } else {
            const double2 a = f[fast::lo_idx<M, CFG>(q, r)], b = f[fast::hi_idx<M, CFG>(q, qm, r)];
            xa = c1 * (a.x + b.x);
            xb = c1 * (a.y - b.y);
            ya = c1 * (a.y + b.y);
            yb = c1 * (b.x - a.x);
          }
          const int64_t ia = j0 ? 0 : j + 1, ib = j0 ? 1 : j + H;
          put<false, EPI>(A, Q.bx + ia, xa, acc);
          put<false, EPI>(A, Q.bx + ib, xb, acc);
          if (has_y) {
            put<false, EPI>(A, Q.by + ia, ya, acc);
            put<false, EPI>(A, Q.by + ib, yb, acc);
          }
        }
      }
    }
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

template <int M>
fpk::Entry make_group(int kind, bool epi) {
  fpk::Entry e;
  switch (kind) {
    case K_SYNTH: e.fn = group_pass<M, K_SYNTH, false>; break;
    case K_ANALYZE: e.fn = epi ? group_pass<M, K_ANALYZE, true> : group_pass<M, K_ANALYZE, false>; break;
    case K_GRAM: e.fn = epi ? group_pass<M, K_GRAM, true> : group_pass<M, K_GRAM, false>; break;
    case K_RESID: e.fn = epi ? nullptr : group_pass<M, K_RESID, false>; break;  // no caller fuses an epilogue here
    default: break;
  }
  e.threads = GCfg<M>::T;
  e.smem = GCfg<M>::SMEM;
  e.w = GCfg<M>::NG;
  return e;
}

}  // namespace gpk
}  // namespace fl
