// fp64 complex FFT engine on shared-memory tiles (sm_100a).
//
// A tile holds F fibres of one axis; fibre f occupies tile[f*fs + k],
// k in [0, m).  The engine is a Stockham autosort FFT over a runtime
// mixed-radix plan (radix 8/4/2/3/5 butterflies in registers, any other
// prime through a direct O(R^2) DFT), ping-ponging between two smem buffers.
// Twiddles come from a per-axis table tw[k] = exp(-2 pi i k / m) built on the
// host in extended precision (fl_runtime.cu), read through the read-only path.
//
// sign = -1: forward DFT (numpy/scipy rfft convention); sign = +1: inverse
// without the 1/m factor (scales are folded into the pack/unpack stages).
#pragma once

#include <cuda_runtime.h>

namespace fl {

constexpr int kMaxStages = 40;

struct AxisPlan {
  int m;                    // complex FFT length (= axis extent)
  int nst;                  // number of radix stages
  int radix[kMaxStages];    // product == m
  const double2* tw;        // device table, m entries
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// multiply by (sign * i):  sign=-1 -> -i z ; sign=+1 -> +i z
__device__ __forceinline__ double2 mul_si(double2 z, int sign) {
  return sign < 0 ? make_double2(z.y, -z.x) : make_double2(-z.y, z.x);
}

__device__ __forceinline__ double2 twiddle(const double2* tw, int e, int sign) {
  double2 w = __ldg(tw + e);
  if (sign > 0) w.y = -w.y;
  return w;
}

// ---- in-register DFTs --------------------------------------------------
__device__ __forceinline__ void dft2(double2* v) {
  double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3, int sign) {
  double2 t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = mul_si(csub(a1, a3), sign);
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, t3);
  a3 = csub(t1, t3);
}

__device__ __forceinline__ void dft8(double2* v, int sign) {
  const double r = 0.70710678118654752440;
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4(e0, e1, e2, e3, sign);
  dft4(o0, o1, o2, o3, sign);
  // o_k *= w8^k, w8 = exp(sign * 2 pi i / 8)
  double2 w1 = make_double2(r, sign * r);
  o1 = cmul(o1, w1);
  o2 = mul_si(o2, sign);
  double2 w3 = make_double2(-r, sign * r);
  o3 = cmul(o3, w3);
  v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
}

__device__ __forceinline__ void dft3(double2* v, int sign) {
  const double c = -0.5, s = 0.86602540378443864676;  // cos, sin(2pi/3)
  double2 a0 = v[0], b = cadd(v[1], v[2]), d = csub(v[1], v[2]);
  double2 t = make_double2(a0.x + c * b.x, a0.y + c * b.y);
  double2 u = mul_si(make_double2(s * d.x, s * d.y), sign);  // sign*i*s*(a1-a2)
  v[0] = cadd(a0, b);
  v[1] = cadd(t, u);
  v[2] = csub(t, u);
}

__device__ __forceinline__ void dft5(double2* v, int sign) {
  const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
  const double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;
  double2 a0 = v[0];
  double2 b1 = cadd(v[1], v[4]), b2 = cadd(v[2], v[3]);
  double2 d1 = csub(v[1], v[4]), d2 = csub(v[2], v[3]);
  double2 t1 = make_double2(a0.x + c1 * b1.x + c2 * b2.x, a0.y + c1 * b1.y + c2 * b2.y);
  double2 t2 = make_double2(a0.x + c2 * b1.x + c1 * b2.x, a0.y + c2 * b1.y + c1 * b2.y);
  double2 u1 = mul_si(make_double2(s1 * d1.x + s2 * d2.x, s1 * d1.y + s2 * d2.y), sign);
  double2 u2 = mul_si(make_double2(s2 * d1.x - s1 * d2.x, s2 * d1.y - s1 * d2.y), sign);
  v[0] = cadd(a0, cadd(b1, b2));
  v[1] = cadd(t1, u1);
  v[4] = csub(t1, u1);
  v[2] = cadd(t2, u2);
  v[3] = csub(t2, u2);
}

// One Stockham butterfly of radix R (compile-time) reading in[r*nb] and
// writing out[r*Ns].
template <int R>
__device__ __forceinline__ void bfly(const double2* __restrict__ in, int nb, double2* __restrict__ out,
                                     int Ns, int j, int tws, const double2* tw, int sign) {
  double2 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = in[r * nb];
  if (j) {
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], twiddle(tw, r * j * tws, sign));
  }
  if constexpr (R == 2) dft2(v);
  else if constexpr (R == 3) dft3(v, sign);
  else if constexpr (R == 4) dft4(v[0], v[1], v[2], v[3], sign);
  else if constexpr (R == 5) dft5(v, sign);
  else if constexpr (R == 8) dft8(v, sign);
#pragma unroll
  for (int r = 0; r < R; ++r) out[r * Ns] = v[r];
}

// Any radix (prime or not): direct DFT, O(R^2) twiddle-table reads.
static __device__ __noinline__ void bfly_any(const double2* __restrict__ in, int nb, double2* __restrict__ out,
                                      int Ns, int j, int tws, int R, int m, const double2* tw,
                                      int sign) {
  const int step = m / R;  // tw[step * e] = exp(-2 pi i e / R)
  for (int k = 0; k < R; ++k) {
    double2 acc = make_double2(0.0, 0.0);
    for (int r = 0; r < R; ++r) {
      double2 v = in[r * nb];
      if (j && r) v = cmul(v, twiddle(tw, r * j * tws, sign));
      const int e = (int)(((long long)r * k) % R);
      acc = cadd(acc, cmul(v, twiddle(tw, e * step, sign)));
    }
    out[k * Ns] = acc;
  }
}

// Batched FFT of the F fibres in ``src`` using ``dst`` as the ping-pong
// buffer; returns the buffer holding the result.  All threads of the block
// participate; ends with __syncthreads().
__device__ __forceinline__ double2* fft_tile(double2* src, double2* dst, int F, int fs,
                                             const AxisPlan& P, int sign) {
  const int m = P.m;
  int Ns = 1;
  for (int s = 0; s < P.nst; ++s) {
    const int R = P.radix[s];
    const int nb = m / R;
    const int tws = m / (Ns * R);
    const int total = F * nb;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const int f = idx % F, q = idx / F;
      const int j = q % Ns;
      const double2* in = src + f * fs + q;
      double2* out = dst + f * fs + (q - j) * R + j;
      switch (R) {
        case 8: bfly<8>(in, nb, out, Ns, j, tws, P.tw, sign); break;
        case 4: bfly<4>(in, nb, out, Ns, j, tws, P.tw, sign); break;
        case 2: bfly<2>(in, nb, out, Ns, j, tws, P.tw, sign); break;
        case 3: bfly<3>(in, nb, out, Ns, j, tws, P.tw, sign); break;
        case 5: bfly<5>(in, nb, out, Ns, j, tws, P.tw, sign); break;
        default: bfly_any(in, nb, out, Ns, j, tws, R, m, P.tw, sign); break;
      }
    }
    __syncthreads();
    double2* t = src;
    src = dst;
    dst = t;
    Ns *= R;
  }
  return src;
}

}  // namespace fl
