// Register-resident axis passes (kernel templates; instantiated per length in fl_fp_*.cu) for power-of-two fibre lengths 16..8192
// (the hot path at every BASELINE size).  Same data model and fusion as the
// generic passes in fl_pass.cu (paired fibres, pack/unpack + ortho scale in
// the load/store stages, one fused last-axis synth+mask+analysis pass, KKT
// epilogue in the final store), with the FFT held in registers:
//
//   synthesis   global rows (j+1, j+h) -> unpack -> smem -> registers ->
//               inverse FFT (NST-1 smem exchanges) -> registers -> global
//   analysis    global -> registers -> forward FFT -> smem -> pack -> global
//   gram/resid  unpack -> inverse FFT -> mask (in registers) -> forward FFT
//               (consumes the inverse FFT's register layout directly) -> pack
//
// A persistent grid (resident CTAs x 148 SMs) walks the tiles.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <string>
#include <type_traits>

#include "fl_common.cuh"
#include "fl_fast.cuh"
#include "fl_mirror.cuh"
#include "fl_internal.h"
#include "fl_passargs.cuh"

namespace fl {
namespace fpk {

using fast::Geom;
using fast::si;
using fast::cfg_code;
using fast::cp_async16;
using fast::cp_async8;
using fast::cp_commit;
using fast::cp_wait;

template <bool STRIDED>
__device__ __forceinline__ void lane_map(int tid, int W, int P, int& c, int& q) {
  if (STRIDED) { c = tid % W; q = tid / W; }  // fibre-fast: 128-byte row segments per quarter-warp
  else { q = tid % P; c = tid / P; }          // position-fast: contiguous rows
}

// Contiguous layout with P = 64 threads per fibre (m = 512, E = 8): place q and
// its pack partner 64 - q in the SAME warp so Z_{m-k} arrives by shuffle.
//   warp A: lanes 0..15 -> q 0..15, lane 16 -> q 32, lanes 17..31 -> q 49..63
//   warp B: lanes 0..15 -> q 16..31, lanes 16..31 -> q 33..48
// partner lane: warp A (lane == 0 || lane == 16) ? lane : 32 - lane; warp B 31 - lane.
__device__ __forceinline__ void lane_map_pair64(int tid, int& c, int& q, int& partner) {
  c = tid >> 6;
  const int l = tid & 63, w = l >> 5, lane = l & 31;
  if (w == 0) {
    q = lane < 16 ? lane : (lane == 16 ? 32 : 32 + lane);
    partner = (lane == 0 || lane == 16) ? lane : 32 - lane;
  } else {
    q = lane < 16 ? 16 + lane : 17 + lane;
    partner = 31 - lane;
  }
}

__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// 16-byte KKT epilogue for a strided-axis pair (x at v, y at v + 1).
__device__ __forceinline__ void kkt_store2(const PassArgs& A, int64_t v, double gx, double gy,
                                           double& acc) {
  const double2 pb = *reinterpret_cast<const double2*>(A.epi.pb + v);
  const double2 pz = *reinterpret_cast<const double2*>(A.epi.pz + v);
  const double2 s1 = *reinterpret_cast<const double2*>(A.epi.sig1 + v);
  const double2 s2 = *reinterpret_cast<const double2*>(A.epi.sig2 + v);
  double2 top, bot;
  {
    const double l1 = add(s1.x, s2.x), l2 = sub(s1.x, s2.x);
    top.x = add(add(gx, mul(l1, pb.x)), mul(l2, pz.x));
    bot.x = add(mul(l2, pb.x), mul(l1, pz.x));
  }
  {
    const double l1 = add(s1.y, s2.y), l2 = sub(s1.y, s2.y);
    top.y = add(add(gy, mul(l1, pb.y)), mul(l2, pz.y));
    bot.y = add(mul(l2, pb.y), mul(l1, pz.y));
  }
  *reinterpret_cast<double2*>(A.out + v) = top;
  if (A.epi.bottom) *reinterpret_cast<double2*>(A.epi.bottom + v) = bot;
  acc += pb.x * top.x + pz.x * bot.x + pb.y * top.y + pz.y * bot.y;
}

// Raw input tile staging: element (k, fibre c) of the tile.
template <int M, bool STRIDED, int CFG>
__device__ __forceinline__ int stage_idx(int k, int c) {
  return STRIDED ? k * Geom<M, CFG>::W + c : c * M + k;
}

// Issue this thread's cp.async copies of tile ``tile`` (its natural-layout
// elements k = q + r P of fibre c) into ``st``.
template <int M, bool STRIDED, int CFG>
__device__ __forceinline__ void issue_tile(const PassArgs& A, int64_t tile, double2* st, int c, int q) {
  using G = Geom<M, CFG>;
  const int64_t g = tile * G::W + c;
  if (g >= A.G) return;
  const Geo Q = geo<STRIDED>(A, g);
#pragma unroll
  for (int r = 0; r < G::E; ++r) {
    const int k = q + r * G::P;
    if (STRIDED) {
      cp_async16(st + stage_idx<M, STRIDED, CFG>(k, c), A.in + Q.bx + k * Q.st);
    } else {
      // planar rows (x row then y row of the pair): conflict-free 8-byte fills
      double* row = reinterpret_cast<double*>(st) + 2 * c * M;
      cp_async8(row + k, A.in + Q.bx + k);
      if (Q.by >= 0) cp_async8(row + M + k, A.in + Q.by + k);
    }
  }
}

// Contiguous axis: the tile's W row pairs as 2W TMA bulk copies (4 KiB rows at
// m = 512) into the planar stage, issued by one thread, completing on ``bar``.
template <int M, int CFG>
__device__ __forceinline__ void tma_tile(const PassArgs& A, int64_t tile, double2* st, unsigned long long* bar,
                                         const double* src = nullptr) {
  if (!src) src = A.in;
  using G = Geom<M, CFG>;
  unsigned bytes = 0;
#pragma unroll 1
  for (int c = 0; c < G::W; ++c) {
    const int64_t g = tile * G::W + c;
    if (g < A.G) bytes += (geo<false>(A, g).by >= 0 ? 2u : 1u) * M * 8u;
  }
  fast::mbar_expect_tx(bar, bytes);
#pragma unroll 1
  for (int c = 0; c < G::W; ++c) {
    const int64_t g = tile * G::W + c;
    if (g >= A.G) break;
    const Geo Q = geo<false>(A, g);
    double* row = reinterpret_cast<double*>(st) + 2 * c * M;
    fast::bulk_g2s(row, src + Q.bx, M * 8u, bar);
    if (Q.by >= 0) fast::bulk_g2s(row + M, src + Q.by, M * 8u, bar);
  }
}

// Element (k, c) of the current raw tile: from staging (pipelined) or global.
template <int M, bool STRIDED, bool PIPE, int CFG>
__device__ __forceinline__ double2 raw(const PassArgs& A, const double2* st, const Geo& Q, bool valid,
                                       int k, int c) {
  double2 z = make_double2(0.0, 0.0);
  if (!valid) return z;
  if (PIPE) {
    if (STRIDED) {
      z = st[stage_idx<M, STRIDED, CFG>(k, c)];
    } else {
      const double* row = reinterpret_cast<const double*>(st) + 2 * c * M;
      z.x = row[k];
      z.y = Q.by < 0 ? 0.0 : row[M + k];
    }
  } else if (STRIDED) {
    z = *reinterpret_cast<const double2*>(A.in + Q.bx + (int64_t)k * Q.st);
  } else {
    z.x = A.in[Q.bx + k];
    if (Q.by >= 0) z.y = A.in[Q.by + k];
  }
  return z;
}

// Single-buffer staging: once every thread has read the current tile out of
// the stage, start copying the next tile into it (overlaps this tile's FFT).
template <int M, bool STRIDED, int CFG>
__device__ __forceinline__ void refill(const PassArgs& A, int64_t next, int64_t ntiles, double2* stage,
                                       int c, int q, unsigned long long* bar = nullptr) {
  if constexpr (Geom<M, CFG>::PIPE == 1) {
    __syncthreads();
    if (bar) {
      if (threadIdx.x == 0 && next < ntiles) tma_tile<M, CFG>(A, next, stage, bar);
      return;
    }
    if (next < ntiles) issue_tile<M, STRIDED, CFG>(A, next, stage, c, q);
    cp_commit();
  }
}

template <int M, bool STRIDED, int KIND, bool EPI, int CFG>
__global__ void __launch_bounds__(Geom<M, CFG>::T, Geom<M, CFG>::MB) fast_pass(const PassArgs A) {
  using G = Geom<M, CFG>;
  constexpr int E = G::E, P = G::P, W = G::W, H = M / 2;
  constexpr int PIPE = G::PIPE;  // 0 none, 1 single, 2 double buffered staging
  extern __shared__ double2 smem[];
  __shared__ double red[32];
  // pack partner by warp shuffle (contiguous layout, 64 threads per fibre)
  constexpr bool SHFL_PACK = !STRIDED && P == 64 && E == 8;
  int c, q, partner = 0;
  if constexpr (SHFL_PACK) lane_map_pair64(threadIdx.x, c, q, partner);
  else lane_map<STRIDED>(threadIdx.x, W, P, c, q);
  double2* fib = smem + c * G::FS;
  double2* stage0 = smem + G::FIB_BYTES / 16;
  double2* stage1 = stage0 + W * M;
  const double2* tw = A.plan.tw;
  const double c0 = A.c0, c1 = A.c1;
  double acc = 0.0, nrm = 0.0;
  const int64_t ntiles = (A.G + W - 1) / W;
  // contiguous rows with single staging: TMA bulk row copies on an mbarrier
  // (one issuing thread, no per-thread cp.async, conflict-free planar fills)
  // The residual pass (K_RESID) also stages its b_hat rows: issued at the top
  // of each tile on a second barrier into a second planar stage, consumed
  // after the inverse FFT (the loads no longer wait behind it).
  __shared__ unsigned long long tbar[2];
  unsigned long long* bar = nullptr;
  unsigned tphase = 0, bphase = 0;
  constexpr bool BSTAGE = KIND == K_RESID && !STRIDED && PIPE == 1;
  const double* bstage = reinterpret_cast<const double*>(stage0 + W * M);
  if constexpr (!STRIDED && PIPE == 1) {
    if ((reinterpret_cast<uintptr_t>(A.in) & 15) == 0 && (!BSTAGE || (reinterpret_cast<uintptr_t>(A.bhat) & 15) == 0)) {
      bar = tbar;
      if (threadIdx.x == 0) {
        fast::mbar_init(bar, 1);
        if (BSTAGE) fast::mbar_init(bar + 1, 1);
      }
      __syncthreads();
    }
  }
  if (PIPE > 0) {
    if (bar) {
      if (threadIdx.x == 0 && (int64_t)blockIdx.x < ntiles) tma_tile<M, CFG>(A, blockIdx.x, stage0, bar);
    } else {
      if ((int64_t)blockIdx.x < ntiles) issue_tile<M, STRIDED, CFG>(A, blockIdx.x, stage0, c, q);
      cp_commit();
    }
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int64_t g = tile * W + c;
    const bool valid = g < A.G;
    const Geo Q = geo<STRIDED>(A, valid ? g : 0);
    const int64_t next = tile + gridDim.x;
    const double2* st = (PIPE == 2 && (it & 1)) ? stage1 : stage0;
    if (BSTAGE && bar && threadIdx.x == 0)  // previous tile's b_hat reads ended at its last barrier
      tma_tile<M, CFG>(A, tile, stage0 + W * M, bar + 1, A.bhat);
    if (PIPE == 2) {
      if (next < ntiles) issue_tile<M, STRIDED, CFG>(A, next, (it & 1) ? stage0 : stage1, c, q);
      cp_commit();
      cp_wait<1>();
      __syncthreads();
    } else if (PIPE == 1) {
      if (bar) {
        fast::mbar_wait(bar, tphase);
        tphase ^= 1u;
      } else {
        cp_wait<0>();
        __syncthreads();
      }
    }
    double2 v[E];
    if (KIND == K_ANALYZE) {
      if (PIPE > 0) {
#pragma unroll
        for (int r = 0; r < E; ++r) v[r] = raw<M, STRIDED, (PIPE > 0), CFG>(A, st, Q, valid, q + r * P, c);
        refill<M, STRIDED, CFG>(A, next, ntiles, stage0, c, q, bar);
      } else {
        // base pointer of row q, rows advance by P*st (no per-element 64-bit multiplies)
        const double* px = A.in + Q.bx + (int64_t)q * Q.st;
        const double* py = A.in + Q.by + (int64_t)q * Q.st;
        const int64_t rs = (int64_t)P * Q.st;
#pragma unroll
        for (int r = 0; r < E; ++r) {
          double2 z = make_double2(0.0, 0.0);
          if (valid) {
            if (STRIDED) z = *reinterpret_cast<const double2*>(px + r * rs);
            else {
              z.x = px[r * rs];
              if (Q.by >= 0) z.y = py[r * rs];
            }
          }
          v[r] = z;
        }
      }
      fast::fft<M, CFG>(v, fib, q, tw, -1);
    } else {
      if constexpr (PIPE > 0) {
        // unpack straight from the staged raw rows into the natural layout:
        // Zin_k needs rows (k+1, k+h) for k < h and rows (M-k+1, M-k+h) above h
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int k = q + r * P;
          double2 z;
          if (r < E / 2) {
            if (r == 0 && q == 0) {
              const double2 a = raw<M, STRIDED, (PIPE > 0), CFG>(A, st, Q, valid, 0, c);
              z = make_double2(c0 * a.x, c0 * a.y);
            } else {
              const double2 a = raw<M, STRIDED, (PIPE > 0), CFG>(A, st, Q, valid, k + 1, c);
              const double2 b = raw<M, STRIDED, (PIPE > 0), CFG>(A, st, Q, valid, k + H, c);
              z = make_double2(c1 * (a.x - b.y), c1 * (b.x + a.y));
            }
          } else {
            if (r == E / 2 && q == 0) {
              const double2 a = raw<M, STRIDED, (PIPE > 0), CFG>(A, st, Q, valid, 1, c);
              z = make_double2(c0 * a.x, c0 * a.y);
            } else {
              const int j = M - k;
              const double2 a = raw<M, STRIDED, (PIPE > 0), CFG>(A, st, Q, valid, j + 1, c);
              const double2 b = raw<M, STRIDED, (PIPE > 0), CFG>(A, st, Q, valid, j + H, c);
              z = make_double2(c1 * (a.x + b.y), c1 * (a.y - b.x));
            }
          }
          v[r] = z;
        }
        refill<M, STRIDED, CFG>(A, next, ntiles, stage0, c, q, bar);
      } else {
        // unpack packed rows (j+1, j+h) into the combined half spectra Zin_j, Zin_{M-j}
        const int qm = -q + ((-q) >> 3);
  #pragma unroll
        for (int r = 0; r < E / 2; ++r) {
          const int j = q + r * P;
          const bool j0 = r == 0 && q == 0;
          const double2 a = raw<M, STRIDED, (PIPE > 0), CFG>(A, st, Q, valid, j0 ? 0 : j + 1, c);
          const double2 b = raw<M, STRIDED, (PIPE > 0), CFG>(A, st, Q, valid, j0 ? 1 : j + H, c);
          const double xa = a.x, ya = a.y, xb = b.x, yb = b.y;
          if (j0) {
            fib[0] = make_double2(c0 * xa, c0 * ya);
            fib[si(H)] = make_double2(c0 * xb, c0 * yb);
          } else {
            fib[fast::lo_idx<M, CFG>(q, r)] = make_double2(c1 * (xa - yb), c1 * (xb + ya));
            fib[fast::hi_idx<M, CFG>(q, qm, r)] = make_double2(c1 * (xa + yb), c1 * (ya - xb));
          }
        }
        __syncthreads();
        fast::load_natural<M, CFG>(v, fib, q);
        __syncthreads();
      }
      // mask words for this thread's samples, fetched before the inverse FFT so
      // their latency hides behind it (one 32-bit word per sample, L1/L2 hits)
      uint32_t wx[(KIND == K_GRAM || KIND == K_RESID) ? E : 1];
      uint32_t wy[(KIND == K_GRAM || KIND == K_RESID) ? E : 1];
      if constexpr (KIND == K_GRAM || KIND == K_RESID) {
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int64_t vx = Q.bx + q + r * P;
          wx[r] = valid ? __ldg(A.bits + (vx >> 5)) : 0u;
          wy[r] = (valid && Q.by >= 0) ? __ldg(A.bits + ((Q.by + q + r * P) >> 5)) : 0u;
        }
      }
      fast::fft<M, CFG>(v, fib, q, tw, +1);
      if (KIND == K_SYNTH) {
        if (valid) {
          double* px = A.out + Q.bx + (int64_t)q * Q.st;
          double* py = A.out + Q.by + (int64_t)q * Q.st;
          const int64_t rs = (int64_t)P * Q.st;
#pragma unroll
          for (int r = 0; r < E; ++r) {
            if (STRIDED) *reinterpret_cast<double2*>(px + r * rs) = v[r];
            else {
              px[r * rs] = v[r].x;
              if (Q.by >= 0) py[r * rs] = v[r].y;
            }
          }
        }
      } else {
        // Z (b_hat - x) or Z x on the synthesized samples, in registers
        if (BSTAGE && bar) {
          fast::mbar_wait(bar + 1, bphase);
          bphase ^= 1u;
        }
        const double* brow = bstage + 2 * c * M;
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int t = q + r * P;
          double2 z = v[r];
          if (valid) {
            const int64_t vx = Q.bx + t;
            const bool mx = (wx[r] >> (vx & 31)) & 1u;
            if (KIND == K_RESID) z.x = mx ? 0.0 : ((BSTAGE && bar) ? brow[t] : A.bhat[vx]) - z.x;
            else if (mx) z.x = 0.0;
            if (Q.by >= 0) {
              const int64_t vy = Q.by + t;
              const bool my = (wy[r] >> (vy & 31)) & 1u;
              if (KIND == K_RESID) z.y = my ? 0.0 : ((BSTAGE && bar) ? brow[M + t] : A.bhat[vy]) - z.y;
              else if (my) z.y = 0.0;
            } else {
              z.y = 0.0;
            }
            if (KIND == K_GRAM) nrm += z.x * z.x + z.y * z.y;  // ||Z A beta||^2 = beta . G beta
          }
          v[r] = z;
        }
        fast::fft<M, CFG>(v, fib, q, tw, -1);
      }
    }
    if (KIND != K_SYNTH && SHFL_PACK) {
      // thread q holds Z_{q + 64 r}; its mirror Z_{512 - q - 64 r} is slot 7 - r of
      // lane `partner` (q = 32: itself, slot 7 - r; q = 0: itself, slot (8 - r) & 7)
      double2 mir[E / 2];
#pragma unroll
      for (int r = 0; r < E / 2; ++r) {
        const double2 sh = shfl2(v[E - 1 - r], partner);
        mir[r] = q == 0 ? v[(E - r) & (E - 1)] : sh;
      }
      if (valid) {
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
          put<STRIDED, EPI>(A, Q.bx + ia, xa, acc);
          put<STRIDED, EPI>(A, Q.bx + ib, xb, acc);
          if (Q.by >= 0) {
            put<STRIDED, EPI>(A, Q.by + ia, ya, acc);
            put<STRIDED, EPI>(A, Q.by + ib, yb, acc);
          }
        }
      }
    } else if (KIND != K_SYNTH) {
      fast::store_natural<M, CFG>(v, fib, q);
      __syncthreads();
      if (valid) {
        const int qm = -q + ((-q) >> 3);
#pragma unroll
        for (int r = 0; r < E / 2; ++r) {
          const int j = q + r * P;
          const bool j0 = r == 0 && q == 0;
          double xa, xb, ya, yb;
          if (j0) {
            const double2 z0 = fib[0], zh = fib[si(H)];
            xa = c0 * z0.x; ya = c0 * z0.y;
            xb = c0 * zh.x; yb = c0 * zh.y;
          } else {
            const double2 a = fib[fast::lo_idx<M, CFG>(q, r)], b = fib[fast::hi_idx<M, CFG>(q, qm, r)];
            xa = c1 * (a.x + b.x);
            xb = c1 * (a.y - b.y);
            ya = c1 * (a.y + b.y);
            yb = c1 * (b.x - a.x);
          }
          const int64_t ia = Q.st * (j0 ? 0 : j + 1), ib = Q.st * (j0 ? 1 : j + H);
          if (STRIDED && !EPI) {
            *reinterpret_cast<double2*>(A.out + Q.bx + ia) = make_double2(xa, ya);
            *reinterpret_cast<double2*>(A.out + Q.bx + ib) = make_double2(xb, yb);
          } else if (STRIDED) {
            kkt_store2(A, Q.bx + ia, xa, ya, acc);
            kkt_store2(A, Q.bx + ib, xb, yb, acc);
          } else {
            put<STRIDED, EPI>(A, Q.bx + ia, xa, acc);
            put<STRIDED, EPI>(A, Q.bx + ib, xb, acc);
            if (Q.by >= 0) {
              put<STRIDED, EPI>(A, Q.by + ia, ya, acc);
              put<STRIDED, EPI>(A, Q.by + ib, yb, acc);
            }
          }
        }
      }
    }
    __syncthreads();
  }
  if (PIPE > 0) cp_wait<0>();
  if (EPI && A.epi.partials) {
    const double s = block_reduce(acc, SumOp(), red);
    if (threadIdx.x == 0) A.epi.partials[blockIdx.x] = s;
  }
  if (KIND == K_GRAM && A.nrm_partials) {
    const double s = block_reduce(nrm, SumOp(), red);
    if (threadIdx.x == 0) A.nrm_partials[blockIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------
// Mirrored-butterfly passes (fl_mirror.cuh) for M = 8^k: the pack and unpack
// read the mirror partner from the thread's own registers, so a pass needs only
// the NST-1 inter-stage shared-memory exchanges.
// ---------------------------------------------------------------------------
template <int M, bool STRIDED, int KIND, bool EPI, int PIPE, int MB = 2, int TT = 0>
__global__ void __launch_bounds__(mirror::MGeom<M, TT>::T, MB) mirror_pass(const PassArgs A) {
  using G = mirror::MGeom<M, TT>;
  // staging geometry shared with Geom<M, CFG> (512-thread CTAs: T_SEL 1)
  constexpr int CFG = G::T == 512 ? cfg_code(1, PIPE, 1, 1) : cfg_code(0, PIPE, 2, 1);
  static_assert(Geom<M, CFG>::P == G::P && Geom<M, CFG>::W == G::W, "staging geometry mismatch");
  static_assert(Geom<M, CFG>::PIPE == PIPE, "staging does not fit");
  constexpr int P = G::P, W = G::W, H = G::H;
  extern __shared__ double2 smem[];
  __shared__ double red[32];
  int c, q;
  lane_map<STRIDED>(threadIdx.x, W, P, c, q);
  const bool q0 = q == 0;
  double2* fib = smem + c * G::FS;
  double2* stage0 = smem + G::FIB_BYTES / 16;
  const double2* tw = A.plan.tw;
  const double c0 = A.c0, c1 = A.c1;
  double acc = 0.0, nrm = 0.0;
  const int64_t ntiles = (A.G + W - 1) / W;
  if (PIPE > 0) {
    if ((int64_t)blockIdx.x < ntiles) issue_tile<M, STRIDED, CFG>(A, blockIdx.x, stage0, c, q);
    cp_commit();
  }
  // strided fused mask pass: when a tile's 8 pairs (16 voxels) share one mask
  // word per row k (row stride a multiple of 32 voxels), the tile's M words are
  // staged in shared memory by the whole CTA (2 words per thread) instead of 16
  // word loads per thread held in registers across the inverse FFT
  // (run_pass_n sends strided fused passes only with A.inner % 32 == 0)
  constexpr bool SMASK = STRIDED && KIND == K_GRAM;
  uint32_t* mw = reinterpret_cast<uint32_t*>(smem + G::FIB_BYTES / 16);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t g = tile * W + c;
    const bool valid = g < A.G;
    const Geo Q = geo<STRIDED>(A, valid ? g : 0);
    const int64_t next = tile + gridDim.x;
    // the fused gram addresses its strided rows at 32-bit element offsets from
    // the pair's base (k * st < 2^32: the launcher refuses larger fibres), so
    // no 64-bit row address stays live across its two FFTs (fewer spills at
    // the 128-register cap: 0.79 -> 0.78 ms at 512^3; the one-FFT passes
    // measured slower with it and keep 64-bit offsets)
    using Off = std::conditional_t<KIND == K_GRAM, uint32_t, int64_t>;
    const double* bin = A.in + Q.bx;
    double* bout = A.out + Q.bx;
    const Off st32 = (Off)Q.st;
    auto ld = [&](int k) -> double2 {
      if constexpr (STRIDED && PIPE == 0) {
        // strided rows bypass L1 (no reuse; it stays with the spill slots of the
        // 128-register FFTs): fused gram 0.775 -> 0.769 ms, analysis axis 1 at
        // 512^3 0.385 -> 0.371 ms, 1024^3 matvec 32.36 -> 32.20 ms
        // ld.global.cg with a 256-byte L2 fetch: the neighbouring tile's half
        // of each 256-byte row segment (the next CTA's) arrives with this one
        // (512^3 matvec 3.133 -> 3.116 ms; neutral at 1024^3)
        double2 z = make_double2(0.0, 0.0);
        if (valid)
          asm volatile("ld.global.cg.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(z.x), "=d"(z.y)
                       : "l"(bin + (Off)k * st32));
        return z;
      } else {
        return raw<M, STRIDED, (PIPE > 0), CFG>(A, stage0, Q, valid, k, c);
      }
    };
    if constexpr (SMASK) {  // the previous tile's reads ended at its forward FFT's first barrier
      const Geo Q0 = geo<STRIDED>(A, tile * W);
      const uint32_t* wb = A.bits + (Q0.bx >> 5);
      const int64_t wst = Q0.st >> 5;
      for (int k = threadIdx.x; k < M; k += G::T) mw[k] = __ldg(wb + k * wst);
    }
    if (PIPE > 0) {
      cp_wait<0>();
      __syncthreads();
    }
    double2 v[16];
    if (KIND == K_ANALYZE) {
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int s = 0; s < 8; ++s)
          v[8 * b + s] = ld(mirror::slot_k<M>(q, b, s));
    } else {
      // Zin_j and Zin_{M-j} from ONE read of the packed rows (j+1, j+H) of
      // j = min(k, M-k); the two values land in the mirror slot pair.
      auto lo = [&](const double2& a, const double2& bb) {  // Zin_j
        return make_double2(c1 * (a.x - bb.y), c1 * (bb.x + a.y));
      };
      auto hi = [&](const double2& a, const double2& bb) {  // Zin_{M-j}
        return make_double2(c1 * (a.x + bb.y), c1 * (a.y - bb.x));
      };
      // Eight row-pair reads per thread, the same code for every lane (a
      // branch on q == 0 would serialise that warp's loads): q = 0 owns the
      // self-mirrored butterflies 0 and NB/2, handled by index / value
      // selects -- rows (0, 1) hold Z_0, Z_H unscaled-paired, its b = 1
      // butterfly starts at NB/2, and its hi values land in other slots.
      constexpr int NB = G::NB;
      const int jb1 = q0 ? NB / 2 : NB - q;
      // hi value i goes to slot GEN[i] (q != 0) or Q0[i] (q == 0); both maps
      // are permutations of the same 8 slots, so two selects per value keep
      // nothing extra live: each slot is written once under either regime.
      constexpr int GEN[8] = {15, 14, 13, 12, 4, 5, 6, 7};
      constexpr int Q0[8] = {4, 7, 6, 5, 12, 13, 14, 15};
      fast::static_for<0, 8>([&](auto I) {
        constexpr int i = decltype(I)::value;
        const int j = i < 4 ? q + i * NB : jb1 + (7 - i) * NB;
        const bool sp = i == 0 && q0;
        double2 a, bb;
        a = ld(sp ? 0 : j + 1);
        bb = ld(sp ? 1 : j + H);
        double2 l = lo(a, bb), h = hi(a, bb);
        if constexpr (i == 0) {
          l = sp ? make_double2(c0 * a.x, c0 * a.y) : l;
          h = sp ? make_double2(c0 * bb.x, c0 * bb.y) : h;
        }
        if constexpr (i < 4) v[i] = l;
        else v[15 - i] = l;
        v[GEN[i]] = q0 ? v[GEN[i]] : h;
        v[Q0[i]] = q0 ? h : v[Q0[i]];
      });
    }
    refill<M, STRIDED, CFG>(A, next, ntiles, stage0, c, q);
    if constexpr (STRIDED && PIPE == 0 && M == 1024) {
      // m = 1024 (one 512-thread CTA per SM): the next tile's M row segments
      // (W pairs x 16 B each) into L2 while this tile runs its FFT, so DRAM
      // keeps streaming through the compute phase.  Only at short strides
      // (axis 1 of 1024^3: 8 KiB, the tile spans one 8 MiB block): 4.75 ->
      // 4.16 ms (synthesis), 4.83 -> 4.01 ms (analysis); at the 8 MiB stride of
      // axis 0 it measured neutral, and at m = 512 (two CTAs per SM) slower.
      if ((next + 1) * W <= A.G && ((A.inner >> 1) % W) == 0) {
        const Geo Qn = geo<STRIDED>(A, next * W);
        if (Qn.st <= (int64_t(1) << 16)) {
          for (int k = threadIdx.x; k < M; k += G::T)
            fast::bulk_prefetch_l2(A.in + Qn.bx + (int64_t)k * Qn.st, W * 16u);
        }
      }
    }
    // mask bits of the 16 slots (x: bit 2i, y: bit 2i+1) packed into one
    // register before the inverse FFT, so no mask word stays live across it
    uint32_t mbits = 0;
    if constexpr ((KIND == K_GRAM || KIND == K_RESID) && !STRIDED && P == 32) {
      // one warp = one row pair of 512 samples = 2 x 16 mask words: lane l
      // loads word l & 15 of row x (l < 16) or row y, slots fetch theirs by
      // shuffle (one live register instead of 32 in-flight word loads)
      const int l = threadIdx.x & 31;
      uint32_t word = 0;
      if (valid && (l < 16 || Q.by >= 0)) word = __ldg(A.bits + (((l < 16) ? Q.bx : Q.by) >> 5) + (l & 15));
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int t = mirror::slot_k<M>(q, i >> 3, i & 7);
        const uint32_t wx = __shfl_sync(0xffffffffu, word, t >> 5);
        const uint32_t wy = __shfl_sync(0xffffffffu, word, 16 + (t >> 5));
        mbits |= ((wx >> (t & 31)) & 1u) << (2 * i);
        mbits |= ((wy >> (t & 31)) & 1u) << (2 * i + 1);
      }
    } else if constexpr ((KIND == K_GRAM || KIND == K_RESID) && !SMASK) {
      if (valid) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int64_t t = mirror::slot_k<M>(q, i >> 3, i & 7);
          const int64_t vx = Q.bx + t * Q.st;
          mbits |= ((__ldg(A.bits + (vx >> 5)) >> (vx & 31)) & 1u) << (2 * i);
          if (Q.by >= 0) {
            const int64_t vy = Q.by + t * Q.st;
            mbits |= ((__ldg(A.bits + (vy >> 5)) >> (vy & 31)) & 1u) << (2 * i + 1);
          }
        }
      }
    }
    // twiddle loads are loop invariant; laundering the table pointer per FFT
    // keeps the compiler from hoisting/CSE-ing them into ~100 live registers
    const double2* tw1 = tw;
    asm volatile("" : "+l"(tw1));
    if (KIND == K_ANALYZE) {
      mirror::fft<M>(v, fib, q, tw1, -1);
    } else {
      mirror::fft<M>(v, fib, q, tw1, +1);
      if (KIND == K_SYNTH) {
        if (valid) {
#pragma unroll
          for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int s = 0; s < 8; ++s) {
              const int64_t t = mirror::slot_k<M>(q, b, s);
              if (STRIDED) *reinterpret_cast<double2*>(bout + (Off)t * st32) = v[8 * b + s];
              else {
                A.out[Q.bx + t] = v[8 * b + s].x;
                if (Q.by >= 0) A.out[Q.by + t] = v[8 * b + s].y;
              }
            }
        }
      } else {
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            double2 z = v[8 * b + s];
            if (valid) {
              const int64_t t = mirror::slot_k<M>(q, b, s);
              const int64_t vx = Q.bx + t * Q.st;
              bool mx, my;
              if constexpr (SMASK) {  // x and y bits of this pair in the tile row's word
                const uint32_t w = mw[t] >> (Q.bx & 31);
                mx = w & 1u;
                my = (w >> 1) & 1u;
              } else {
                mx = (mbits >> (2 * (8 * b + s))) & 1u;
                my = (mbits >> (2 * (8 * b + s) + 1)) & 1u;
              }
              if (KIND == K_RESID) z.x = mx ? 0.0 : A.bhat[vx] - z.x;
              else if (mx) z.x = 0.0;
              if (Q.by >= 0) {
                const int64_t vy = Q.by + t * Q.st;
                if (KIND == K_RESID) z.y = my ? 0.0 : A.bhat[vy] - z.y;
                else if (my) z.y = 0.0;
              } else {
                z.y = 0.0;
              }
              // (the strided gram serves only the KKT apply, never the PCG norm)
              if (KIND == K_GRAM && !STRIDED) nrm += z.x * z.x + z.y * z.y;
            }
            v[8 * b + s] = z;
          }
        const double2* tw2 = tw;
        asm volatile("" : "+l"(tw2));
        mirror::fft<M>(v, fib, q, tw2, -1);
      }
    }
    if (KIND != K_SYNTH && valid) {
      // pack (Z_k, Z_{M-k}) straight from registers for the 8 slots with k < H
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int j = mirror::slot_k<M>(q, b, s);
          const double2 a = v[8 * b + s];
          double xa, xb, ya, yb;
          Off ia, ib;
          if (b == 0 && s == 0 && q0) {
            const double2 zh = v[4];  // Z_H of q = 0
            xa = c0 * a.x; ya = c0 * a.y;
            xb = c0 * zh.x; yb = c0 * zh.y;
            ia = 0;
            ib = st32;
          } else {
            // mirror partner of slot (b, s) (indices are constants after unrolling)
            const double2 m = q0 ? v[8 * b + (b == 0 ? ((8 - s) & 7) : (7 - s))] : v[8 * (1 - b) + 7 - s];
            xa = c1 * (a.x + m.x);
            xb = c1 * (a.y - m.y);
            ya = c1 * (a.y + m.y);
            yb = c1 * (m.x - a.x);
            ia = st32 * (Off)(j + 1);
            ib = st32 * (Off)(j + H);
          }
          if (STRIDED && !EPI) {
            *reinterpret_cast<double2*>(bout + ia) = make_double2(xa, ya);
            *reinterpret_cast<double2*>(bout + ib) = make_double2(xb, yb);
          } else if (STRIDED) {
            kkt_store2(A, Q.bx + ia, xa, ya, acc);
            kkt_store2(A, Q.bx + ib, xb, yb, acc);
          } else {
            put<STRIDED, EPI>(A, Q.bx + ia, xa, acc);
            put<STRIDED, EPI>(A, Q.bx + ib, xb, acc);
            if (Q.by >= 0) {
              put<STRIDED, EPI>(A, Q.by + ia, ya, acc);
              put<STRIDED, EPI>(A, Q.by + ib, yb, acc);
            }
          }
        }
    }
  }
  if (PIPE > 0) cp_wait<0>();
  if (EPI && A.epi.partials) {
    const double s = block_reduce(acc, SumOp(), red);
    if (threadIdx.x == 0) A.epi.partials[blockIdx.x] = s;
  }
  if (KIND == K_GRAM && A.nrm_partials) {
    const double s = block_reduce(nrm, SumOp(), red);
    if (threadIdx.x == 0) A.nrm_partials[blockIdx.x] = s;
  }
}

struct Entry {
  KernelFn fn = nullptr;
  int threads = 0, smem = 0, w = 0;
};

// One kernel per (length, strided, kind, epilogue), no run-time switches.
// Variant choice (measured in round 1 with per-pass CUDA events, DESIGN 4.1):
//   * plain strided synthesis / analysis ("light"): the mirrored engine for
//     m = 64 / 512 / 4096 (fl_mirror.cuh, 256 threads, no staging), else the
//     E = 8 engine on 512-thread CTAs without staging (2 CTAs/SM);
//   * everything else at m <= 512: 256-thread CTAs with single-buffer
//     staging; m >= 1024: the same with one CTA per SM and the full register
//     budget (E = 16);
//   * contiguous m = 512 / 1024 / 2048 passes and every strided m = 1024
//     stride are dispatched before this table (fl_gpass.cuh, fl_wpass.cuh,
//     fl_mirror.cuh fft1024).
constexpr int kCfgLight = cfg_code(1, 0, 2);
constexpr int kCfgHeavy = cfg_code(0, 1, 2);
constexpr int kCfgLong = cfg_code(0, 1, 1);

template <int M, bool S, int CFG>
Entry entry_of(KernelFn fn) {
  Entry e;
  using G = Geom<M, CFG>;
  e.fn = fn;
  e.threads = G::T;
  e.smem = G::SMEM;
  e.w = G::W;
  return e;
}

template <int M, bool S, int CFG>
Entry make_heavy(int kind, bool epi) {
  using G = Geom<M, CFG>;
  if (kind == K_SYNTH) return entry_of<M, S, CFG>(fast_pass<M, S, K_SYNTH, false, CFG>);
  if (kind == K_ANALYZE) {
    if constexpr (S) return epi ? Entry() : entry_of<M, S, CFG>(fast_pass<M, S, K_ANALYZE, false, CFG>);
    else return entry_of<M, S, CFG>(epi ? fast_pass<M, S, K_ANALYZE, true, CFG> : fast_pass<M, S, K_ANALYZE, false, CFG>);
  }
  if constexpr (!S) {
    if (kind == K_GRAM)
      return entry_of<M, S, CFG>(epi ? fast_pass<M, S, K_GRAM, true, CFG> : fast_pass<M, S, K_GRAM, false, CFG>);
    if (kind == K_RESID) {
      if (epi) return Entry();  // no caller fuses an epilogue into the residual pass
      Entry e = entry_of<M, S, CFG>(fast_pass<M, S, K_RESID, false, CFG>);
      if (G::PIPE == 1) e.smem += G::STAGE_BYTES;  // the staged b_hat rows
      return e;
    }
  }
  return Entry();
}

template <int M, bool S>
Entry make(int kind, bool epi) {
  const bool light = S && !epi && (kind == K_SYNTH || kind == K_ANALYZE);
  if constexpr (S && (M == 64 || M == 512 || M == 4096)) {
    if (light) {
      using G = mirror::MGeom<M>;
      Entry e;
      e.fn = kind == K_SYNTH ? mirror_pass<M, true, K_SYNTH, false, 0> : mirror_pass<M, true, K_ANALYZE, false, 0>;
      e.threads = G::T;
      e.smem = G::FIB_BYTES;
      e.w = G::W;
      return e;
    }
  }
  if constexpr (S && M == 512) {
    // strided fused gram: the mask pass of the axis-0-last operator order
    // (op_gram, KKT apply at 512^3) on the mirrored engine, the tile's mask
    // words staged in shared memory
    if (kind == K_GRAM && !epi) {
      using G = mirror::MGeom<M>;
      Entry e;
      e.fn = mirror_pass<M, true, K_GRAM, false, 0>;
      e.threads = G::T;
      e.smem = G::FIB_BYTES + M * 4;
      e.w = G::W;
      return e;
    }
  }
  if constexpr (S && M <= 512 && !(M == 64 || M == 512)) {
    if (light) {
      return entry_of<M, S, kCfgLight>(kind == K_SYNTH ? fast_pass<M, S, K_SYNTH, false, kCfgLight>
                                                       : fast_pass<M, S, K_ANALYZE, false, kCfgLight>);
    }
  }
  if constexpr (M == 1024 && S) return Entry();  // dispatched to the mirrored engine (make_mirror1024)
  else if constexpr (M >= 1024) return make_heavy<M, S, kCfgLong>(kind, epi);
  else return make_heavy<M, S, kCfgHeavy>(kind, epi);
}

// strided m = 1024 synthesis / analysis on the mirrored 8 x 16 x 8 engine
// (512-thread CTAs: 8 fibre pairs = 128-byte row segments, one CTA per SM)
template <int M = 1024>  // a template: instantiated only in the TU that uses it
Entry make_mirror1024(int kind) {
  using G = mirror::MGeom<M>;
  Entry e;
  e.fn = kind == K_SYNTH ? mirror_pass<M, true, K_SYNTH, false, 0, 1>
                         : mirror_pass<M, true, K_ANALYZE, false, 0, 1>;
  e.threads = G::T;
  e.smem = G::FIB_BYTES;
  e.w = G::W;
  return e;
}

template <int M>
Entry make_any(bool strided, int kind, bool epi) {
  return strided ? make<M, true>(kind, epi) : make<M, false>(kind, epi);
}

}  // namespace fpk
}  // namespace fl
