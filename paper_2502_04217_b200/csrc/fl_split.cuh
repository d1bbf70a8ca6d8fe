// Strided synthesis / analysis passes for m = 1024 as two mirrored 512-point
// FFTs per fibre pair (the C5 axes).
//
// The generic E = 16 engine needs ~200 registers at m = 1024 (one 8-warp CTA
// per SM).  Here the length-1024 transform is split once by radix 2 and each
// half runs on the mirrored-butterfly engine of fl_mirror.cuh (128 registers):
//
//   synthesis (inverse, DIT):  E = IDFT512(Zin_even), O = IDFT512(Zin_odd),
//       z[n] = E[n] + w^n O[n],  z[n + 512] = E[n] - w^n O[n],  w = e^{+2 pi i/1024}
//   analysis (forward, DIF):   a[n] = z[n] + z[n + 512],  b[n] = (z[n] - z[n + 512]) w^n,
//       X[2k] = DFT512(a)[k],  X[2k + 1] = DFT512(b)[k],  w = e^{-2 pi i/1024}
//
// A tile is W = 8 fibre pairs (128-byte row segments on the strided axis) x
// two halves x 32 lanes = 512 threads, fibre-fast lanes as in the mirrored
// 512 passes.  Half h = 0 ("A") owns the even spectrum / first time half,
// h = 1 ("B") the odd spectrum / second time half; lane q of both halves owns
// the same 512-point slot positions j = own(q, b) + 64 s, so the radix-2
// combine is one shared-memory swap between the halves.  Real-pair packing:
// Z_{2j} pairs with Z_{1024-2j} = Z_{2(512-j)} (A's own mirror slot, in
// registers); Z_{2j+1} pairs with Z_{2(511-j)+1} (B, read back through
// shared memory).
#pragma once

#include "fl_mirror.cuh"
#include "fl_passargs.cuh"

namespace fl {
namespace split {

using G = mirror::MGeom<512>;    // NB = 64, P = 32 lanes per half
constexpr int M = 1024, H = 512;  // transform length, packing half
constexpr int W = 8;              // fibre pairs per tile
constexpr int T = W * 2 * G::P;   // 512 threads
constexpr int SMEM = W * 2 * G::FS * 16;

__device__ __forceinline__ double2 row(const PassArgs& A, const Geo& Q, bool valid, int r) {
  return valid ? *reinterpret_cast<const double2*>(A.in + Q.bx + (int64_t)r * Q.st) : make_double2(0.0, 0.0);
}

// Zin_k of the packed rows (fourier.py:176-181 inverse), k in [0, 1024).
__device__ __forceinline__ double2 zin(const PassArgs& A, const Geo& Q, bool valid, int k) {
  const double c0 = A.c0, c1 = A.c1;
  if (k == 0 || k == H) {
    const double2 a = row(A, Q, valid, k == 0 ? 0 : 1);
    return make_double2(c0 * a.x, c0 * a.y);
  }
  const int j = k < H ? k : M - k;
  const double2 a = row(A, Q, valid, j + 1), b = row(A, Q, valid, j + H);
  return k < H ? make_double2(c1 * (a.x - b.y), c1 * (b.x + a.y)) : make_double2(c1 * (a.x + b.y), c1 * (a.y - b.x));
}

__device__ __forceinline__ void put2(const PassArgs& A, const Geo& Q, int r, double x, double y) {
  *reinterpret_cast<double2*>(A.out + Q.bx + (int64_t)r * Q.st) = make_double2(x, y);
}

// pack (Z_k, Z_{M-k}) into rows (k+1, k+H); k = 0 -> rows (0, 1) from Z_0, Z_H
__device__ __forceinline__ void pack(const PassArgs& A, const Geo& Q, int k, double2 a, double2 m) {
  const double c1 = A.c1;
  put2(A, Q, k + 1, c1 * (a.x + m.x), c1 * (a.y + m.y));
  put2(A, Q, k + H, c1 * (a.y - m.y), c1 * (m.x - a.x));
}

template <int KIND>
__global__ void __launch_bounds__(T, 1) split_pass(const PassArgs A) {
  extern __shared__ double2 smem[];
  const int tid = threadIdx.x;
  const int c = tid % W, rest = tid / W;  // fibre-fast: 8 lanes cover one 128-byte row segment
  const int h = rest / G::P, q = rest % G::P;
  const bool q0 = q == 0;
  double2* fib = smem + (c * 2 + h) * G::FS;
  const double2* oth = smem + (c * 2 + (1 - h)) * G::FS;
  const double2* tw = A.plan.tw;  // length-1024 table e^{-2 pi i t / 1024}
  const int64_t ntiles = (A.G + W - 1) / W;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t g = tile * W + c;
    const bool valid = g < A.G;
    const Geo Q = geo<true>(A, valid ? g : 0);
    double2 v[16];
    if constexpr (KIND == K_SYNTH) {
      if (h == 0) {
        // even spectrum: slot j holds Zin_{2j}, its mirror slot 512 - j holds
        // Zin_{1024-2j} -- one read of rows (2j+1, 2j+512) serves both (the
        // mirrored unpack of fl_fastpass.cuh with k = 2j); q = 0 owns Z_0, Z_H
        const double c0 = A.c0, c1 = A.c1;
        constexpr int NB = G::NB;
        const int jb1 = q0 ? NB / 2 : NB - q;
        constexpr int GEN[8] = {15, 14, 13, 12, 4, 5, 6, 7};
        constexpr int Q0[8] = {4, 7, 6, 5, 12, 13, 14, 15};
        fast::static_for<0, 8>([&](auto I) {
          constexpr int i = decltype(I)::value;
          const int j = i < 4 ? q + i * NB : jb1 + (7 - i) * NB;  // 512-space index, j < 256
          const bool sp = i == 0 && q0;
          const double2 a = row(A, Q, valid, sp ? 0 : 2 * j + 1);
          const double2 bb = row(A, Q, valid, sp ? 1 : 2 * j + H);
          double2 l = make_double2(c1 * (a.x - bb.y), c1 * (bb.x + a.y));  // Zin_{2j}
          double2 hh = make_double2(c1 * (a.x + bb.y), c1 * (a.y - bb.x));  // Zin_{1024-2j}
          if constexpr (i == 0) {
            l = sp ? make_double2(c0 * a.x, c0 * a.y) : l;
            hh = sp ? make_double2(c0 * bb.x, c0 * bb.y) : hh;
          }
          if constexpr (i < 4) v[i] = l;
          else v[15 - i] = l;
          v[GEN[i]] = q0 ? v[GEN[i]] : hh;
          v[Q0[i]] = q0 ? hh : v[Q0[i]];
        });
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = zin(A, Q, valid, 2 * mirror::slot_k<512>(q, i >> 3, i & 7) + 1);
      }
      mirror::fft<512, 0, 1024>(v, fib, q, tw, +1);
      // radix-2 combine: swap E / O between the halves through shared memory
#pragma unroll
      for (int i = 0; i < 16; ++i) fib[fast::si(mirror::slot_k<512>(q, i >> 3, i & 7))] = v[i];
      __syncthreads();
      if (valid) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j = mirror::slot_k<512>(q, i >> 3, i & 7);
          const double2 other = oth[fast::si(j)];
          const double2 e = h == 0 ? v[i] : other;
          const double2 wo = cmul(twiddle(tw, j, +1), h == 0 ? other : v[i]);
          const double2 z = h == 0 ? cadd(e, wo) : csub(e, wo);
          *reinterpret_cast<double2*>(A.out + Q.bx + (int64_t)(j + h * H) * Q.st) = z;
        }
      }
      __syncthreads();  // the next tile's exchanges reuse fib
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int j = mirror::slot_k<512>(q, i >> 3, i & 7);
        const double2 z0 = row(A, Q, valid, j), z1 = row(A, Q, valid, j + H);
        v[i] = h == 0 ? cadd(z0, z1) : cmul(csub(z0, z1), twiddle(tw, j, -1));
      }
      mirror::fft<512, 0, 1024>(v, fib, q, tw, -1);
      // B publishes its outputs: Z_{2j+1} pairs with B's slot 511 - j of another lane
      if (h == 1) {
#pragma unroll
        for (int i = 0; i < 16; ++i) fib[fast::si(mirror::slot_k<512>(q, i >> 3, i & 7))] = v[i];
      }
      __syncthreads();
      if (valid) {
        const double c0 = A.c0;
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int s = 0; s < 4; ++s) {  // the slots with j < 256 write
            const int j = mirror::slot_k<512>(q, b, s);
            const double2 a = v[8 * b + s];
            if (h == 0) {
              if (b == 0 && s == 0 && q0) {  // Z_0 and Z_H (slot (0, 4) of q = 0 holds j = 256)
                const double2 zh = v[4];
                put2(A, Q, 0, c0 * a.x, c0 * a.y);
                put2(A, Q, 1, c0 * zh.x, c0 * zh.y);
              } else {
                const double2 m = q0 ? v[8 * b + (b == 0 ? ((8 - s) & 7) : (7 - s))] : v[8 * (1 - b) + 7 - s];
                pack(A, Q, 2 * j, a, m);
              }
            } else {
              pack(A, Q, 2 * j + 1, a, fib[fast::si(511 - j)]);
            }
          }
      }
      __syncthreads();
    }
  }
}

}  // namespace split
}  // namespace fl
