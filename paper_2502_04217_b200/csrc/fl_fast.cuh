// Register-resident fp64 FFT engine for power-of-two fibre lengths (sm_100a).
//
// A fibre of length M is owned by P = M/E threads; thread q holds the E
// elements q + r*P (r = 0..E-1) in registers ("natural layout").  Each
// Stockham stage of radix R (R | E) runs B = E/R butterflies per thread in
// registers; between stages the data are exchanged once through shared
// memory (write, sync, read natural layout, sync).  After the last stage the
// registers are back in natural layout, so a forward FFT can consume an
// inverse FFT's output with no exchange (fused gram), and global loads/stores
// of natural-order data go straight to/from registers.
//
// Shared memory index of element k of fibre c: c*FS + k + (k >> 3) with
// FS = M + M/8 + 1 (odd).  With fibre-fast lanes (strided axes) every
// quarter-warp touches 8 fibres at one k -> 8 distinct 16-byte bank groups;
// with position-fast lanes (contiguous axis) the k + k/8 skew spreads the
// stride-R write of the first stage.  Both layouts are conflict-free.
#pragma once

#include <type_traits>

#include "fl_fft.cuh"

namespace fl {
namespace fast {

__device__ __forceinline__ int si(int k) { return k + (k >> 3); }

// Compile-time loop: f(std::integral_constant<int, I>{}) for I in [B, E).
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }
constexpr int nfull(int m, int e) { return (m % e == 0 && m > 1) ? 1 + nfull(m / e, e) : 0; }
constexpr int imax(int a, int b) { return a > b ? a : b; }

// CFG selects the CTA shape, input staging and residency target of a pass
// kernel: CFG = cfg_code(T_SEL, PIPE, MB) with T_SEL 0 -> 256 threads,
// 1 -> 512 threads, MB = CTAs per SM requested from __launch_bounds__, and
//   PIPE 0 -> registers load straight from global (no staging),
//        1 -> one cp.async staging buffer, refilled with the next tile as
//             soon as the current tile has been read out of it,
//        2 -> two staging buffers (double buffering).
constexpr int cfg_code(int t_sel, int pipe, int mb, int e16 = 0) {
  return e16 * 27 + t_sel * 9 + pipe * 3 + (mb - 1);
}

template <int M, int CFG = 0>
struct Geom {
  static constexpr int E = (M >= 1024 || CFG >= 27) ? 16 : 8;   // elements per thread
  static constexpr int P = M / E;                               // threads per fibre
  static constexpr int T_SEL = (CFG % 27) / 9;
  static constexpr int PIPE_REQ = (CFG / 3) % 3;
  static constexpr int MB = CFG % 3 + 1;
  static constexpr int T = imax(T_SEL ? 512 : 256, P);          // threads per CTA
  static constexpr int W = T / P;                               // fibres per CTA tile
  static constexpr int FS = M + M / 8 + 1;                      // smem fibre stride (double2)
  static constexpr int FIB_BYTES = W * FS * 16;                 // exchange buffer
  static constexpr int STAGE_BYTES = W * M * 16;                // one raw input tile
  static constexpr int PIPE = FIB_BYTES + PIPE_REQ * STAGE_BYTES <= 220 * 1024 ? PIPE_REQ : 0;
  static constexpr int SMEM = FIB_BYTES + PIPE * STAGE_BYTES;
  static constexpr int NFULL = nfull(M, E);
  static constexpr int REM = M / ipow(E, NFULL);                // first-stage radix if > 1
  static constexpr int NST = NFULL + (REM > 1 ? 1 : 0);
  static constexpr int radix(int s) { return (REM > 1 && s == 0) ? REM : E; }
  static constexpr int ns(int s) { return s == 0 ? 1 : ns(s - 1) * radix(s - 1); }
};

// ---- cp.async (LDGSTS) helpers ----
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }

// ---- TMA bulk copies (cp.async.bulk) completing on an mbarrier ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// global -> shared bulk copy of ``bytes`` (multiple of 16, both sides 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// Bulk L2 prefetch of ``bytes`` (multiple of 16) at a 16-byte aligned address.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- DFT kernels on register arrays (stride-aware) ----
template <int R, int STRIDE>
__device__ __forceinline__ void dft_gather(double2* v, int sign) {
  double2 t[R];
#pragma unroll
  for (int s = 0; s < R; ++s) t[s] = v[s * STRIDE];
  if constexpr (R == 2) dft2(t);
  else if constexpr (R == 4) dft4(t[0], t[1], t[2], t[3], sign);
  else if constexpr (R == 8) dft8(t, sign);
  else if constexpr (R == 16) {
    // 16 = 4 x 4: four DFT4 on stride-4 subsequences, twiddle, four DFT4
    double2 u[16];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double2 x0 = t[a], x1 = t[a + 4], x2 = t[a + 8], x3 = t[a + 12];
      dft4(x0, x1, x2, x3, sign);
      u[a] = x0; u[a + 4] = x1; u[a + 8] = x2; u[a + 12] = x3;  // u[a + 4*k1]
    }
    // twiddle w16^(a*k1)
    const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
    const double r2 = 0.70710678118654752440;
    const double2 w[10] = {{1, 0}, {c1, sign * s1}, {r2, sign * r2}, {s1, sign * c1}, {0, (double)sign},
                           {-s1, sign * c1}, {-r2, sign * r2}, {-c1, sign * s1}, {-1, 0}, {-c1, -sign * s1}};
#pragma unroll
    for (int a = 1; a < 4; ++a)
#pragma unroll
      for (int k1 = 1; k1 < 4; ++k1) u[a + 4 * k1] = cmul(u[a + 4 * k1], w[a * k1]);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      double2 x0 = u[4 * k1], x1 = u[4 * k1 + 1], x2 = u[4 * k1 + 2], x3 = u[4 * k1 + 3];
      dft4(x0, x1, x2, x3, sign);
      t[k1] = x0; t[k1 + 4] = x1; t[k1 + 8] = x2; t[k1 + 12] = x3;  // X[k1 + 4*k2]
    }
  }
#pragma unroll
  for (int s = 0; s < R; ++s) v[s * STRIDE] = t[s];
}

// Twiddle powers w^s, s = 0..R-1, w = exp(sign 2 pi i j / (Ns R)) from the
// length-M table (3 table reads, the rest by products).
template <int M, int R, int NS>
__device__ __forceinline__ void twiddles(double2* w, int j, const double2* tw, int sign) {
  constexpr int step = M / (NS * R);
  w[0] = make_double2(1.0, 0.0);
  if constexpr (R >= 2) w[1] = twiddle(tw, j * step, sign);
  if constexpr (R >= 4) {
    w[2] = twiddle(tw, 2 * j * step, sign);
    w[3] = cmul(w[1], w[2]);
  }
  if constexpr (R >= 8) {
    w[4] = twiddle(tw, 4 * j * step, sign);
    w[5] = cmul(w[1], w[4]);
    w[6] = cmul(w[2], w[4]);
    w[7] = cmul(w[3], w[4]);
  }
  if constexpr (R >= 16) {
    const double2 w8 = twiddle(tw, 8 * j * step, sign);
#pragma unroll
    for (int s = 8; s < 16; ++s) w[s] = cmul(w[s - 8], w8);
  }
}

// One stage: butterflies of radix R on the natural-layout registers.
template <int M, int CFG, int S>
__device__ __forceinline__ void stage_compute(double2* v, int q, const double2* tw, int sign) {
  using G = Geom<M, CFG>;
  constexpr int R = G::radix(S), NS = G::ns(S), B = G::E / R, P = G::P;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    if constexpr (NS > 1) {
      const int j = (q + b * P) % NS;
      double2 w[R];
      twiddles<M, R, NS>(w, j, tw, sign);
#pragma unroll
      for (int s = 1; s < R; ++s) v[b + s * B] = cmul(v[b + s * B], w[s]);
    }
    dft_gather<R, B>(v + b, sign);
  }
}

// Write stage S outputs to smem at their Stockham destinations.  The padded
// index si(pos) is split into a per-butterfly base plus compile-time offsets
// wherever the stage geometry allows it (no per-element integer math).
template <int M, int CFG, int S>
__device__ __forceinline__ void stage_store(const double2* v, double2* fib, int q) {
  using G = Geom<M, CFG>;
  constexpr int R = G::radix(S), NS = G::ns(S), B = G::E / R, P = G::P;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int qq = q + b * P;
    if constexpr (NS % 8 == 0) {
      const int j = qq % NS;
      double2* o = fib + si((qq - j) * R + j);
#pragma unroll
      for (int s = 0; s < R; ++s) o[s * (NS + NS / 8)] = v[b + s * B];
    } else if constexpr (NS == 1 && R == 8) {
      double2* o = fib + 9 * qq;  // si(8 qq + s) = 9 qq + s
#pragma unroll
      for (int s = 0; s < R; ++s) o[s] = v[b + s * B];
    } else {
      const int j = qq % NS;
      const int base = (qq - j) * R + j;
#pragma unroll
      for (int s = 0; s < R; ++s) fib[si(base + s * NS)] = v[b + s * B];
    }
  }
}

// Natural layout: element q + r P.  For P % 8 == 0, si(q + r P) = si(q) + r (P + P/8).
template <int M, int CFG>
__device__ __forceinline__ void load_natural(double2* v, const double2* fib, int q) {
  using G = Geom<M, CFG>;
  constexpr int P = G::P;
  if constexpr (P % 8 == 0) {
    const double2* o = fib + si(q);
#pragma unroll
    for (int r = 0; r < G::E; ++r) v[r] = o[r * (P + P / 8)];
  } else {
#pragma unroll
    for (int r = 0; r < G::E; ++r) v[r] = fib[si(q + r * P)];
  }
}

template <int M, int CFG>
__device__ __forceinline__ void store_natural(const double2* v, double2* fib, int q) {
  using G = Geom<M, CFG>;
  constexpr int P = G::P;
  if constexpr (P % 8 == 0) {
    double2* o = fib + si(q);
#pragma unroll
    for (int r = 0; r < G::E; ++r) o[r * (P + P / 8)] = v[r];
  } else {
#pragma unroll
    for (int r = 0; r < G::E; ++r) fib[si(q + r * P)] = v[r];
  }
}

// si(j) and si(M - j) for j = q + r P (r < E/2): per-thread part + constants.
// With a = M - r P (a multiple of 8 when P is): si(a - q) = a + a/8 + qm,
// qm = -q + floor(-q / 8).
template <int M, int CFG>
__device__ __forceinline__ int lo_idx(int q, int r) {
  constexpr int P = Geom<M, CFG>::P;
  if constexpr (P % 8 == 0) return si(q) + r * (P + P / 8);
  else return si(q + r * P);
}
template <int M, int CFG>
__device__ __forceinline__ int hi_idx(int q, int qm, int r) {
  constexpr int P = Geom<M, CFG>::P;
  if constexpr (P % 8 == 0) return (M - r * P) + (M - r * P) / 8 + qm;
  else return si(M - q - r * P);
}

// Full FFT from natural-layout registers to natural-layout registers.
template <int M, int CFG, int S = 0>
__device__ __forceinline__ void fft(double2* v, double2* fib, int q, const double2* tw, int sign) {
  using G = Geom<M, CFG>;
  stage_compute<M, CFG, S>(v, q, tw, sign);
  if constexpr (S + 1 < G::NST) {
    stage_store<M, CFG, S>(v, fib, q);
    __syncthreads();
    load_natural<M, CFG>(v, fib, q);
    __syncthreads();
    fft<M, CFG, S + 1>(v, fib, q, tw, sign);
  }
}

}  // namespace fast
}  // namespace fl
