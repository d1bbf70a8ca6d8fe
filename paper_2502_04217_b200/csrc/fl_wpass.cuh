// Two-stage warp-owned contiguous-axis passes (fibre length 1024; the
// template also covers 512, where the group passes of fl_gpass.cuh win).
//
// The CTA-tiled and group-decoupled engines run a 512-point FFT as three
// radix-8 stages with two shared-memory exchanges; a fused gram pass (inverse
// FFT, mask, forward FFT) then moves every element through shared memory four
// times, and at 512^3 that made the pass L1/shared-bound (89.6 % L1/TEX busy,
// profiles/r02_gram512_group_ncu.md).  Here m = E x P with E = 32 elements per
// thread and P = m / 32 threads per fibre pair (16 at m = 512: two pairs per
// warp; 32 at m = 1024: one pair per warp), and each FFT is two in-register
// stages with ONE exchange between them:
//
//   inverse (synthesis), input k = q + P r (thread q, slot r):
//     DFT_32 over r in registers, twiddle w_m^(q k1), exchange (buf[k1][q]),
//     DFT_P over q for k1 in {q' + P j}: output t = k1 + 32 k2 in slot (j, k2)
//   forward (analysis) from that layout, t = a + 32 b:
//     DFT_P over b in registers, twiddle w_m^(-a f1), exchange (buf[a][f1]),
//     DFT_32 over a: output f = f1 + P f2 in slot f2 of thread f1 -- natural.
//
// Analysis loads its rows straight into the split layout, synthesis stores
// straight from it, so every pass kind has one exchange per FFT and the fused
// gram two instead of four; both exchanges use the
// same padded layout (row stride P + 1 double2), conflict-free for the column
// writes and row reads of the first and the row writes and column reads of
// the second.  A pair never leaves its warp: __syncwarp only, no named or CTA
// barriers.  The real-pair unpack and pack (fourier.py:176-181, :193-197) use
// the mirror symmetry of the natural layout: slot r of thread q holds
// k = q + P r, whose mirror m - k is slot 31 - r of thread P - q (thread 0:
// its own slot 32 - r), so each packed row value is loaded once and the
// partner values travel by warp shuffle.  Rows are read straight from global
// memory (coalesced 8-byte loads along the row; staging them through TMA cost
// two of the eight warps per SM and was slower); the mask bits of the fused
// pass (masking.py:107-118) come from one word per lane, gathered by shuffle.
#pragma once

#include "fl_fastpass.cuh"

namespace fl {
namespace wpk {

// CTAs per SM asked of __launch_bounds__ (one: 255 registers for the 32 elements per thread)
constexpr int kWpMinBlocks = 1;

// cos / sin(2 pi m / 32), m = 0..31
__device__ __forceinline__ constexpr double c32(int m) {
  constexpr double t[32] = {
      1.0, 0.98078528040323044913, 0.92387953251128675613, 0.83146961230254523708,
      0.70710678118654752440, 0.55557023301960222474, 0.38268343236508977173, 0.19509032201612826785,
      0.0, -0.19509032201612826785, -0.38268343236508977173, -0.55557023301960222474,
      -0.70710678118654752440, -0.83146961230254523708, -0.92387953251128675613, -0.98078528040323044913,
      -1.0, -0.98078528040323044913, -0.92387953251128675613, -0.83146961230254523708,
      -0.70710678118654752440, -0.55557023301960222474, -0.38268343236508977173, -0.19509032201612826785,
      0.0, 0.19509032201612826785, 0.38268343236508977173, 0.55557023301960222474,
      0.70710678118654752440, 0.83146961230254523708, 0.92387953251128675613, 0.98078528040323044913};
  return t[m & 31];
}
__device__ __forceinline__ constexpr double s32(int m) { return c32(m - 8); }  // sin x = cos(x - pi/2)

// In-register DFT of 32 natural-order values (sign * 2 pi i convention of fl_fft.cuh):
// 32 = 8 x 4: DFT_8 on the stride-4 subsequences, twiddle w32^(a k1), DFT_4 over a.
template <int STRIDE>
__device__ __forceinline__ void dft32(double2* v, int sign) {
  double2 u[32];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double2 t[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) t[i] = v[(a + 4 * i) * STRIDE];
    dft8(t, sign);
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) {
      const int m = a * k1;
      if (m == 0) {
        u[a + 4 * k1] = t[k1];
      } else {
        const double2 w = make_double2(c32(m), sign * s32(m));
        u[a + 4 * k1] = cmul(t[k1], w);
      }
    }
  }
#pragma unroll
  for (int k1 = 0; k1 < 8; ++k1) {
    double2 x0 = u[4 * k1], x1 = u[4 * k1 + 1], x2 = u[4 * k1 + 2], x3 = u[4 * k1 + 3];
    dft4(x0, x1, x2, x3, sign);
    v[(k1) * STRIDE] = x0;
    v[(k1 + 8) * STRIDE] = x1;
    v[(k1 + 16) * STRIDE] = x2;
    v[(k1 + 24) * STRIDE] = x3;
  }
}

template <int N, int STRIDE>
__device__ __forceinline__ void dftn(double2* v, int sign) {
  if constexpr (N == 32) dft32<STRIDE>(v, sign);
  else fast::dft_gather<N, STRIDE>(v, sign);
}

// v[k * STRIDE] *= w_M^(sign * base * k), k = 1..N-1 (N <= 32), from five
// table powers: w^(base k) = w^(4 base m) w^(base l) for k = 4m + l, each
// factor at most two products from a table entry (~3 ulp).  The bases are
// loop invariant; the compiler keeps what it can of the powers across pairs.
template <int M, int N, int STRIDE>
__device__ __forceinline__ void twiddle_run(double2* v, int base, const double2* tw, int sign) {
  double2 p1[4], p4[8];
  p1[0] = make_double2(1.0, 0.0);
  p1[1] = twiddle(tw, base, sign);
  p1[2] = twiddle(tw, 2 * base, sign);
  p1[3] = cmul(p1[1], p1[2]);
  p4[0] = make_double2(1.0, 0.0);
  if constexpr (N > 4) {
    p4[1] = twiddle(tw, 4 * base, sign);
    p4[2] = twiddle(tw, 8 * base, sign);
    p4[3] = cmul(p4[1], p4[2]);
  }
  if constexpr (N > 16) {
    p4[4] = twiddle(tw, 16 * base, sign);
    p4[5] = cmul(p4[1], p4[4]);
    p4[6] = cmul(p4[2], p4[4]);
    p4[7] = cmul(p4[3], p4[4]);
  }
#pragma unroll
  for (int k = 1; k < N; ++k) {
    const int m = k >> 2, l = k & 3;
    const double2 w = m == 0 ? p1[l] : (l == 0 ? p4[m] : cmul(p4[m], p1[l]));
    v[k * STRIDE] = cmul(v[k * STRIDE], w);
  }
}

template <int M>
struct WG {
  static constexpr int E = 32, P = M / 32, PPW = 32 / P;  // pairs per warp
  static constexpr int NJ = E / P;                        // k1 values per thread after the exchange
  static constexpr int SROW = P + 1;                      // padded row (double2)
  static constexpr int BUF = E * SROW;                    // double2 per pair
  static constexpr int WARPS = 8, T = WARPS * 32, PPC = WARPS * PPW;
  static constexpr int WARP_BYTES = PPW * BUF * 16;
  static constexpr int SMEM = WARPS * WARP_BYTES;
  static constexpr int MINB = kWpMinBlocks;
};

// Inverse FFT: natural layout (slot r = element q + P r) -> slot j * P + k2 =
// element (q + P j) + 32 k2.
template <int M>
__device__ __forceinline__ void inv_fft(double2* v, double2* buf, int q, const double2* tw) {
  using G = WG<M>;
  constexpr int P = G::P, S = G::SROW;
  dft32<1>(v, +1);
  twiddle_run<M, 32, 1>(v, q, tw, +1);
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < 32; ++k1) buf[k1 * S + q] = v[k1];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < G::NJ; ++j) {
#pragma unroll
    for (int qq = 0; qq < P; ++qq) v[j * P + qq] = buf[(q + P * j) * S + qq];
    dftn<P, 1>(v + j * P, +1);
  }
}

// Forward FFT from the inverse's output layout back to the natural layout.
template <int M>
__device__ __forceinline__ void fwd_fft_from_split(double2* v, double2* buf, int q, const double2* tw) {
  using G = WG<M>;
  constexpr int P = G::P, S = G::SROW;
#pragma unroll
  for (int j = 0; j < G::NJ; ++j) {
    dftn<P, 1>(v + j * P, -1);
    twiddle_run<M, P, 1>(v + j * P, q + P * j, tw, -1);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < G::NJ; ++j)
#pragma unroll
    for (int f1 = 0; f1 < P; ++f1) buf[(q + P * j) * S + f1] = v[j * P + f1];
  __syncwarp();
#pragma unroll
  for (int a = 0; a < 32; ++a) v[a] = buf[a * S + q];
  dft32<1>(v, -1);
}

__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// NRM: the fused gram also reduces ||Z A beta||^2 (the PCG curvature); the
// KKT apply's gram skips it (1024^3: 4.70 -> 4.60 ms)
template <int M, int KIND, bool EPI, bool NRM = true>
__global__ void __launch_bounds__(WG<M>::T, WG<M>::MINB) warp_pass(const PassArgs A) {
  using G = WG<M>;
  constexpr int E = G::E, P = G::P, H = M / 2, NJ = G::NJ;
  constexpr bool MASKED = KIND == K_GRAM || KIND == K_RESID;
  extern __shared__ double2 smem[];
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane % P, h = lane / P;       // position in the pair, pair within the warp
  const int lbase = lane - q;                 // first lane of this pair
  const int partner = lbase + ((P - q) & (P - 1));
  const bool q0 = q == 0;
  double2* buf = smem + (warp * G::PPW + h) * G::BUF;
  const double2* tw = A.plan.tw;
  const double c0 = A.c0, c1 = A.c1;
  const int64_t npairs = A.G;
  const int64_t gstride = (int64_t)gridDim.x * G::PPC;
  double acc = 0.0, nrm = 0.0;
  for (int64_t gw = ((int64_t)blockIdx.x * G::WARPS + warp) * G::PPW; gw < npairs; gw += gstride) {
    const int64_t g = gw + h;
    const bool valid = g < npairs;
    const Geo Q = geo<false>(A, valid ? g : gw);
    const bool has_y = Q.by >= 0;
    const double* rx = A.in + Q.bx;
    const double* ry = A.in + Q.by;
    {  // L2 prefetch of the warp's next rows (one 128-byte line per lane and step)
      const int64_t gn = gw + gstride;
      if (gn < npairs) {
        const Geo Qn = geo<false>(A, gn);
        const int64_t nrows = (npairs - gn) < G::PPW ? (npairs - gn) : G::PPW;
        const char* base = reinterpret_cast<const char*>(A.in + Qn.bx);
        const int64_t bytes = (Qn.by >= 0 ? 2 : 1) * nrows * M * 8;
        for (int64_t off = (int64_t)lane * 128; off < bytes; off += 32 * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
      }
    }
    // mask words of the pair (one x and one y word per lane), loaded before the
    // rows so both latencies overlap; the bits are extracted after the unpack
    uint32_t mx = 0, my = 0;
    uint32_t wxl = 0, wyl = 0;
    if constexpr (MASKED) {
      const int wl = lane - lbase;
      if (valid && wl < P) {
        wxl = __ldg(A.bits + (Q.bx >> 5) + wl);
        if (has_y) wyl = __ldg(A.bits + (Q.by >> 5) + wl);
      }
    }
    double2 v[E];
    if constexpr (KIND == K_ANALYZE) {
      // load straight into the split layout the forward FFT starts from:
      // slot (j, b) = element (q + P j) + 32 b (coalesced along the row)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int b = 0; b < P; ++b) {
          const int t = (q + P * j) + 32 * b;
          v[j * P + b] = valid ? make_double2(rx[t], has_y ? ry[t] : 0.0) : make_double2(0.0, 0.0);
        }
    } else {
      // unpack: each packed row value is read once; Zin_k (k < H) stays, Zin_{M-k} goes
      // to the mirror slot (thread P - q, slot 31 - r; thread 0: its own slot 32 - r)
      double2 hi[E / 2];
#pragma unroll
      for (int r = 0; r < E / 2; ++r) {
        const int k = q + P * r;
        const bool edge = q0 && r == 0;
        const int ia = edge ? 0 : k + 1, ib = edge ? 1 : k + H;
        double ax = 0.0, ay = 0.0, bx = 0.0, by = 0.0;
        if (valid) {
          ax = rx[ia];
          bx = rx[ib];
          if (has_y) {
            ay = ry[ia];
            by = ry[ib];
          }
        }
        if (edge) {
          v[0] = make_double2(c0 * ax, c0 * ay);
          hi[0] = make_double2(c0 * bx, c0 * by);  // Zin_H -> thread 0 slot E/2
        } else {
          v[r] = make_double2(c1 * (ax - by), c1 * (bx + ay));
          hi[r] = make_double2(c1 * (ax + by), c1 * (ay - bx));
        }
      }
#pragma unroll
      for (int r = 0; r < E / 2; ++r) {
        const double2 rv = shfl2(hi[r], partner);
        v[E - 1 - r] = rv;  // thread q >= 1: partner's slot r mirrors our slot 31 - r
      }
      if (q0) {  // thread 0 is its own partner: slot 32 - r <- hi[r], slot 16 <- Zin_H
        v[E / 2] = hi[0];
#pragma unroll
        for (int r = 1; r < E / 2; ++r) v[E - r] = hi[r];
      }
    }
    if constexpr (MASKED) {
      // after the inverse FFT slot (j, k2) holds element (q + P j) + 32 k2: word k2, bit q + P j
      if constexpr (P == 32) {
        // 32 x 32 bit transpose by ballot: bit k2 of ballot qt = bit qt of word k2
#pragma unroll
        for (int qt = 0; qt < 32; ++qt) {
          const uint32_t bx = __ballot_sync(0xffffffffu, (wxl >> qt) & 1u);
          const uint32_t by = __ballot_sync(0xffffffffu, (wyl >> qt) & 1u);
          if (q == qt) {
            mx = bx;
            my = by;
          }
        }
      } else {
#pragma unroll
        for (int k2 = 0; k2 < P; ++k2) {
          const uint32_t wx = __shfl_sync(0xffffffffu, wxl, lbase + k2);
          const uint32_t wy = __shfl_sync(0xffffffffu, wyl, lbase + k2);
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            mx |= ((wx >> (q + P * j)) & 1u) << (j * P + k2);
            my |= ((wy >> (q + P * j)) & 1u) << (j * P + k2);
          }
        }
      }
    }
    if constexpr (KIND == K_ANALYZE) {
      fwd_fft_from_split<M>(v, buf, q, tw);
    } else {
      inv_fft<M>(v, buf, q, tw);
      if constexpr (KIND == K_SYNTH) {
        // slot (j, k2) = element (q + P j) + 32 k2
        if (valid) {
#pragma unroll
          for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int k2 = 0; k2 < P; ++k2) {
              const int t = (q + P * j) + 32 * k2;
              A.out[Q.bx + t] = v[j * P + k2].x;
              if (has_y) A.out[Q.by + t] = v[j * P + k2].y;
            }
        }
      } else {
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int k2 = 0; k2 < P; ++k2) {
            const int s = j * P + k2;
            const int t = (q + P * j) + 32 * k2;
            double2 z = v[s];
            const bool bmx = (mx >> s) & 1u, bmy = (my >> s) & 1u;
            if (KIND == K_RESID) {
              z.x = (bmx || !valid) ? 0.0 : __ldg(A.bhat + Q.bx + t) - z.x;
              z.y = (bmy || !has_y || !valid) ? 0.0 : __ldg(A.bhat + Q.by + t) - z.y;
            } else {
              if (bmx || !valid) z.x = 0.0;
              if (bmy || !has_y || !valid) z.y = 0.0;
              if constexpr (NRM) nrm += z.x * z.x + z.y * z.y;  // ||Z A beta||^2 = beta . G beta
            }
            v[s] = z;
          }
        fwd_fft_from_split<M>(v, buf, q, tw);
      }
    }
    if constexpr (KIND != K_SYNTH) {
    // pack: rows (j+1, j+H) from Z_k (slot r < 16) and Z_{M-k} (mirror slot:
    // slot 31 - r of the partner; thread 0: its own slot 32 - r)
    double2 mir[E / 2];
#pragma unroll
    for (int r = 0; r < E / 2; ++r) {
      const double2 sh = shfl2(v[E - 1 - r], partner);
      mir[r] = q0 ? v[(E - r) & (E - 1)] : sh;
    }
    if (valid) {
#pragma unroll
      for (int r = 0; r < E / 2; ++r) {
        const int k = q + P * r;
        const bool j0 = q0 && r == 0;
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
        const int64_t ia = j0 ? 0 : k + 1, ib = j0 ? 1 : k + H;
        put<false, EPI>(A, Q.bx + ia, xa, acc);
        put<false, EPI>(A, Q.bx + ib, xb, acc);
        if (has_y) {
          put<false, EPI>(A, Q.by + ia, ya, acc);
          put<false, EPI>(A, Q.by + ib, yb, acc);
        }
      }
    }
    }  // pack
  }
  if (EPI && A.epi.partials) {
    const double s = block_reduce(acc, SumOp(), red);
    if (threadIdx.x == 0) A.epi.partials[blockIdx.x] = s;
  }
  if (KIND == K_GRAM && NRM && A.nrm_partials) {
    const double s = block_reduce(nrm, SumOp(), red);
    if (threadIdx.x == 0) A.nrm_partials[blockIdx.x] = s;
  }
}

template <int M>
fpk::Entry make_warp(int kind, bool epi, bool nrm) {
  fpk::Entry e;
  switch (kind) {
    case K_SYNTH: e.fn = warp_pass<M, K_SYNTH, false>; break;
    case K_ANALYZE: e.fn = epi ? warp_pass<M, K_ANALYZE, true> : warp_pass<M, K_ANALYZE, false>; break;
    case K_GRAM:
      e.fn = epi ? warp_pass<M, K_GRAM, true> : nrm ? warp_pass<M, K_GRAM, false> : warp_pass<M, K_GRAM, false, false>;
      break;
    case K_RESID: e.fn = epi ? nullptr : warp_pass<M, K_RESID, false>; break;
    default: break;
  }
  e.threads = WG<M>::T;
  e.smem = WG<M>::SMEM;
  e.w = WG<M>::PPC;
  return e;
}

}  // namespace wpk
}  // namespace fl
