// "Mirrored" register FFT engine for M = 8^k (64, 512, 4096), sm_100a.
//
// Every stage is radix 8 with NB = M/8 butterflies per fibre; a fibre is owned
// by P = NB/2 threads and thread q owns the two MIRRORED butterflies
//
//     b = 0 : qq = q              b = 1 : qq = NB - q   (q = 0: qq = NB/2)
//
// Butterfly qq reads positions qq + s*NB and, in the last stage, writes
// qq + s*NB, so slot (b, s) of thread q holds index k = qq_b + s*NB and its
// mirror M - k sits in the SAME thread:
//
//     q != 0 : (b, s) <-> (1 - b, 7 - s)
//     q == 0 : (0, s) <-> (0, (8 - s) mod 8),  (1, s) <-> (1, 7 - s)
//
// so the real-pair pack (Z_k, Z_{M-k}) and the unpack (Zin_k from the packed
// rows of min(k, M-k)) need no shared-memory exchange; only the NST-1
// inter-stage exchanges remain.  Registers: v[b*8 + s].
#pragma once

#include "fl_fast.cuh"

namespace fl {
namespace mirror {

using fast::si;

constexpr int log8(int m) { return m <= 1 ? 0 : 1 + log8(m / 8); }

template <int M, int TT = 0>
struct MGeom {
  static constexpr int E = 16;
  static constexpr int NB = M / 8;                          // butterflies per fibre per stage
  static constexpr int P = NB / 2;                          // threads per fibre
  // threads per CTA: 256 (two CTAs per SM); m = 1024 (64 threads per pair):
  // 512, so a tile is still 8 fibre pairs = 128-byte row segments; TT forces T
  static constexpr int T = TT ? TT : (M == 1024 ? 512 : fast::imax(256, P));
  static constexpr int W = T / P;                           // fibres per CTA tile
  static constexpr int NST = log8(M);
  static constexpr int FS = M + M / 8 + 1;                  // smem fibre stride (double2)
  static constexpr int FIB_BYTES = W * FS * 16;
  static constexpr int STAGE_BYTES = W * M * 16;
  static constexpr int H = M / 2;
  static constexpr int ns(int s) { return s == 0 ? 1 : 8 * ns(s - 1); }
};

__device__ __forceinline__ int own(int q, int b, int nb) { return b == 0 ? q : (q == 0 ? nb / 2 : nb - q); }

// One radix-8 stage on both butterflies (twiddles from a length-TM table,
// TM = M normally; TM = 2M when the length-M FFT is a half of a 2M one).
template <int M, int S, int TM = M>
__device__ __forceinline__ void stage(double2* v, int q, const double2* tw, int sign) {
  using G = MGeom<M>;
  constexpr int NS = G::ns(S);
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    double2* u = v + 8 * b;
    if constexpr (NS > 1) {
      const int qq = own(q, b, G::NB);
      const int j = qq % NS;
      // fast::twiddles' products applied as they are formed (the same values):
      // w1, w2, w4 from the table, w3 = w1 w2, w5 = w1 w4, w6 = w2 w4,
      // w7 = w3 w4, with at most four twiddles live (register pressure of the
      // two-FFT fused passes)
      constexpr int step = TM / (NS * 8);
      const double2 w1 = twiddle(tw, j * step, sign);
      const double2 w2 = twiddle(tw, 2 * j * step, sign);
      const double2 w4 = twiddle(tw, 4 * j * step, sign);
      u[1] = cmul(u[1], w1);
      u[2] = cmul(u[2], w2);
      u[4] = cmul(u[4], w4);
      u[5] = cmul(u[5], cmul(w1, w4));
      u[6] = cmul(u[6], cmul(w2, w4));
      const double2 w3 = cmul(w1, w2);
      u[3] = cmul(u[3], w3);
      u[7] = cmul(u[7], cmul(w3, w4));
    }
    dft8(u, sign);
  }
}

// Exchange after stage S: outputs to their Stockham destinations, then the
// inputs of stage S+1 (positions qq + s*NB of the thread's butterflies).
template <int M, int S>
__device__ __forceinline__ void exchange(double2* v, double2* fib, int q) {
  using G = MGeom<M>;
  constexpr int NS = G::ns(S), NB = G::NB;
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    const int qq = own(q, b, NB);
    if constexpr (NS == 1) {
      double2* o = fib + 9 * qq;  // si(8 qq + s) = 9 qq + s
#pragma unroll
      for (int s = 0; s < 8; ++s) o[s] = v[8 * b + s];
    } else {
      const int j = qq % NS;
      double2* o = fib + si((qq - j) * 8 + j);
#pragma unroll
      for (int s = 0; s < 8; ++s) o[s * (NS + NS / 8)] = v[8 * b + s];
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    const double2* o = fib + si(own(q, b, NB));
#pragma unroll
    for (int s = 0; s < 8; ++s) v[8 * b + s] = o[s * (NB + NB / 8)];
  }
  __syncthreads();
}

// m = 1024 = 8 x 16 x 8: Stockham stages of radix 8 (spans 1), 16 (span 8) and
// 8 (span 128).  The first and last stages have 128 butterflies and keep the
// mirror ownership {q, 128 - q} (so unpack and pack find Z_k and Z_{m-k} in
// the same thread, exactly as for 8^k); the middle radix-16 stage has one
// butterfly per thread (butterfly q: positions q + 64 t).
__device__ __forceinline__ void fft1024(double2* v, double2* fib, int q, const double2* tw, int sign) {
  constexpr int NB = 128;
  const int o0 = own(q, 0, NB), o1 = own(q, 1, NB);
  dft8(v, sign);
  dft8(v + 8, sign);
  {  // stage 0 (span 1): outputs at 8 qq + t, si = 9 qq + t
    double2* a = fib + 9 * o0;
    double2* b = fib + 9 * o1;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      a[t] = v[t];
      b[t] = v[8 + t];
    }
  }
  __syncthreads();
  {  // stage 1 inputs: q + 64 t, si = si(q) + 72 t
    const double2* a = fib + si(q);
#pragma unroll
    for (int t = 0; t < 16; ++t) v[t] = a[72 * t];
  }
  __syncthreads();
  const int j = q & 7;  // span 8: twiddle w128^(j t)
  if (j) {
    double2 w[16];
    fast::twiddles<1024, 16, 8>(w, j, tw, sign);
#pragma unroll
    for (int t = 1; t < 16; ++t) v[t] = cmul(v[t], w[t]);
  }
  fast::dft_gather<16, 1>(v, sign);
  {  // stage 1 outputs: (q - j) 16 + j + 8 t, si = si(base) + 9 t
    double2* a = fib + si((q - j) * 16 + j);
#pragma unroll
    for (int t = 0; t < 16; ++t) a[9 * t] = v[t];
  }
  __syncthreads();
  {  // stage 2 inputs: own + 128 t, si = si(own) + 144 t
    const double2* a = fib + si(o0);
    const double2* b = fib + si(o1);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      v[t] = a[144 * t];
      v[8 + t] = b[144 * t];
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < 2; ++b) {  // stage 2 (span 128): twiddle w1024^(own t), outputs own + 128 t
    const int ob = b ? o1 : o0;
    double2 w[8];
    fast::twiddles<1024, 8, 128>(w, ob, tw, sign);
#pragma unroll
    for (int t = 1; t < 8; ++t) v[8 * b + t] = cmul(v[8 * b + t], w[t]);
    dft8(v + 8 * b, sign);
  }
}

template <int M, int S = 0, int TM = M>
__device__ __forceinline__ void fft(double2* v, double2* fib, int q, const double2* tw, int sign) {
  if constexpr (M == 1024) {
    fft1024(v, fib, q, tw, sign);
    return;
  } else {
  stage<M, S, TM>(v, q, tw, sign);
  if constexpr (S + 1 < MGeom<M>::NST) {
    exchange<M, S>(v, fib, q);
    fft<M, S + 1, TM>(v, fib, q, tw, sign);
  }
  }
}

// Index k held by slot (b, s) of thread q.
template <int M>
__device__ __forceinline__ int slot_k(int q, int b, int s) {
  return own(q, b, MGeom<M>::NB) + s * MGeom<M>::NB;
}

}  // namespace mirror
}  // namespace fl
