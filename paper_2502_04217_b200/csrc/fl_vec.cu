// Elementwise and reduction kernels of the IPM / PCG path (sm_100a).
//
// Compiled with -fmad=false and written with explicit round-to-nearest
// intrinsics in NumPy's left-to-right evaluation order,
// so every elementwise quantity is bitwise identical to the reference on
// equal inputs.  Reductions are two-level (per-block partials in a fixed
// grid, then one block per row in block order): deterministic run to run,
// not bitwise equal to NumPy/OpenBLAS summation.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <string>

#include "fl_common.cuh"
#include "fl_internal.h"

namespace fl {
namespace {

constexpr int T = 256;

__device__ __forceinline__ double nanmax(double a, double b) {
  return (isnan(a) || isnan(b)) ? NAN : fmax(a, b);
}
__device__ __forceinline__ double nanmin(double a, double b) {
  return (isnan(a) || isnan(b)) ? NAN : fmin(a, b);
}
struct NanMaxOp {
  static constexpr double identity = -__builtin_huge_val();
  __device__ double operator()(double a, double b) const { return nanmax(a, b); }
};
struct NanMinOp {
  static constexpr double identity = __builtin_huge_val();
  __device__ double operator()(double a, double b) const { return nanmin(a, b); }
};

template <class Op>
__device__ __forceinline__ void emit(double v, Op op, double* red, double* partials, int row) {
  v = block_reduce(v, op, red);
  if (threadIdx.x == 0) partials[(size_t)row * gridDim.x + blockIdx.x] = v;
}

#define GRID_LOOP(i, n) \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ---------------- masks (masking.py) ----------------
__global__ void k_mask_bits(int64_t n, const uint8_t* __restrict__ flags, uint32_t* __restrict__ bits,
                            int64_t* __restrict__ counts) {
  const int64_t nw = (n + 31) >> 5;
  GRID_LOOP(w, nw) {
    uint32_t word = 0;
    int valid = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t v = (w << 5) + b;
      if (v < n) {
        ++valid;
        if (flags[v]) word |= 1u << b;
      }
    }
    bits[w] = word;
    counts[w] = valid - __popc(word);
  }
}

// Bragg-peak punch (workloads.bragg_flags): voxel missing when the summed
// squared periodic distances to the nearest multiple of `spacing` along every
// axis are <= r2.  Integer distances, compared in double as NumPy does.
__global__ void k_bragg_bits(int64_t n, int ndim, int64_t d1, int64_t d2, int64_t sp, double r2,
                             uint32_t* __restrict__ bits, int64_t* __restrict__ counts) {
  const int64_t nw = (n + 31) >> 5;
  GRID_LOOP(w, nw) {
    uint32_t word = 0;
    int valid = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t v = (w << 5) + b;
      if (v >= n) break;
      ++valid;
      int64_t rem = v, sum = 0;
      const int64_t ext[2] = {d2, d1};
      for (int a = 0; a < ndim; ++a) {  // innermost axis first
        int64_t t;
        if (a < ndim - 1) {
          const int64_t e = ext[a];
          t = rem % e;
          rem /= e;
        } else {
          t = rem;
        }
        t %= sp;
        const int64_t m = t < sp - t ? t : sp - t;
        sum += m * m;
      }
      if ((double)sum <= r2) word |= 1u << b;
    }
    bits[w] = word;
    counts[w] = valid - __popc(word);
  }
}

__device__ __forceinline__ int64_t obs_slot(const uint32_t* bits, const int64_t* off, int64_t v,
                                            bool& miss) {
  const uint32_t word = bits[v >> 5];
  const int b = (int)(v & 31);
  miss = (word >> b) & 1u;
  return off[v >> 5] + __popc(~word & ((1u << b) - 1u));
}

__global__ void k_embed(int64_t n, const uint32_t* __restrict__ bits, const int64_t* __restrict__ off,
                        const double* __restrict__ obs, double* __restrict__ full) {
  GRID_LOOP(v, n) {
    bool miss;
    const int64_t s = obs_slot(bits, off, v, miss);
    full[v] = miss ? 0.0 : obs[s];
  }
}

// Counter-based observation noise for on-device inputs:
// the draw of a voxel is a function of (seed, GLOBAL flat voxel index) only,
// so a full grid, an X-slab and a Y-slab (any rank count) see bitwise the same
// noise.  Local index k -> local coordinates (l0, l1, l2) in the box `ext`;
// global index = sum_a (l_a + off_a) * stride_a.  Two splitmix64 words ->
// Box-Muller (cosine branch), u1 in (0, 1].
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_noisy_embed(int64_t nl, int64_t e1, int64_t e2, int64_t o0, int64_t o1, int64_t o2, int64_t s0,
                              int64_t s1, int64_t s2, uint64_t seed, double sigma,
                              const uint32_t* __restrict__ bits, double* __restrict__ x) {
  GRID_LOOP(k, nl) {
    const bool miss = (bits[k >> 5] >> (k & 31)) & 1u;
    if (miss) {
      x[k] = 0.0;
      continue;
    }
    const int64_t l2 = k % e2, t = k / e2;
    const int64_t l1 = t % e1, l0 = t / e1;
    const uint64_t g = (uint64_t)((l0 + o0) * s0 + (l1 + o1) * s1 + (l2 + o2) * s2);
    const uint64_t h1 = mix64(seed ^ mix64(2 * g)), h2 = mix64(seed ^ mix64(2 * g + 1));
    const double u1 = (double)((h1 >> 11) + 1) * 0x1.0p-53;
    const double u2 = (double)(h2 >> 11) * 0x1.0p-53;
    x[k] = __dadd_rn(x[k], __dmul_rn(sigma, __dmul_rn(sqrt(-2.0 * log(u1)), cospi(2.0 * u2))));
  }
}

__global__ void k_gather(int64_t n, const uint32_t* __restrict__ bits, const int64_t* __restrict__ off,
                         const double* __restrict__ full, double* __restrict__ obs) {
  GRID_LOOP(v, n) {
    bool miss;
    const int64_t s = obs_slot(bits, off, v, miss);
    if (!miss) obs[s] = full[v];
  }
}

// ---------------- barrier diagonals (newton_system.py:72-91) ----------------
__device__ __forceinline__ bool bad(double v) { return !(v > 0.0) || !isfinite(v); }

__global__ void k_diagonals(int64_t n, const double* __restrict__ s1, const double* __restrict__ s2,
                            const double* __restrict__ nu1, const double* __restrict__ nu2,
                            double* __restrict__ sig1, double* __restrict__ sig2,
                            double* __restrict__ lam1, double* __restrict__ lam2,
                            double* __restrict__ dvec, double* __restrict__ bvec,
                            double* __restrict__ partials) {
  __shared__ double red[32];
  double flag = 0.0;
  GRID_LOOP(i, n) {
    const double a = s1[i], b = s2[i], c = nu1[i], d = nu2[i];
    if (bad(a) || bad(b) || bad(c) || bad(d)) flag = 1.0;
    const double g1 = dvd(c, a), g2 = dvd(d, b);
    sig1[i] = g1;
    sig2[i] = g2;
    const double l1 = add(g1, g2);
    if (lam1) lam1[i] = l1;
    if (lam2) lam2[i] = sub(g1, g2);
    const double dv = add(add(g1, g2), mul(mul(4.0, g1), g2));
    if (dvec) dvec[i] = dv;
    if (bvec) bvec[i] = dvd(dv, add(1.0, l1));
  }
  emit(flag, MaxOp(), red, partials, 0);
}

// z = P^{-1} r in NumPy order (newton_system.py:155-159) from sigma1, sigma2.
struct Pinv {
  double l1, l2, dv, bv;
  __device__ __forceinline__ Pinv(double g1, double g2) {
    l1 = add(g1, g2);
    l2 = sub(g1, g2);
    dv = add(add(g1, g2), mul(mul(4.0, g1), g2));
    bv = dvd(dv, add(1.0, l1));
  }
  __device__ __forceinline__ double top(double rb, double rc) const {
    return dvd(sub(mul(l1, rb), mul(l2, rc)), dv);
  }
  __device__ __forceinline__ double bot(double rb, double rc) const {
    return add(mul(dvd(-l2, dv), rb), dvd(rc, bv));
  }
};

__global__ void k_precond(int64_t n, const double* __restrict__ g1, const double* __restrict__ g2,
                          const double* __restrict__ rb, const double* __restrict__ rc,
                          double* __restrict__ top, double* __restrict__ bot) {
  GRID_LOOP(i, n) {
    const Pinv P(g1[i], g2[i]);
    const double a = rb[i], c = rc[i];
    top[i] = P.top(a, c);
    bot[i] = P.bot(a, c);
  }
}

// ---------------- newton_rhs (newton_system.py:113-145) ----------------
__global__ void k_newton_rhs(int64_t n, fl_state st, const double* __restrict__ g,
                             const double* __restrict__ sig1, const double* __restrict__ sig2,
                             double lam, double mu, double* r1o, double* r2o, double* r3o,
                             double* r4o, double* r5o, double* r6o, double* __restrict__ rbo,
                             double* __restrict__ rco) {
  GRID_LOOP(i, n) {
    const double beta = st.beta[i], z = st.z[i], s1 = st.s1[i], s2 = st.s2[i];
    const double y1 = st.y1[i], y2 = st.y2[i];
    const double r1 = sub(add(g[i], y1), y2);
    const double r2 = sub(add(y1, y2), lam);
    const double r3 = sub(y1, dvd(mu, s1));
    const double r4 = sub(y2, dvd(mu, s2));
    const double r5 = sub(add(z, beta), s1);
    const double r6 = sub(sub(z, beta), s2);
    const double g1 = sig1[i], g2 = sig2[i];
    rbo[i] = add(sub(add(sub(r1, r3), r4), mul(g1, r5)), mul(g2, r6));
    rco[i] = sub(sub(sub(sub(r2, r3), r4), mul(g1, r5)), mul(g2, r6));
    if (r1o) r1o[i] = r1;
    if (r2o) r2o[i] = r2;
    if (r3o) r3o[i] = r3;
    if (r4o) r4o[i] = r4;
    if (r5o) r5o[i] = r5;
    if (r6o) r6o[i] = r6;
  }
}

// ---------------- direction recovery (newton_system.py:184-196, ipm.py:334-338) -------
struct Dir {
  double dy1, dy2, ds1c, ds2c;  // condensed convention (recover_eliminated)
  double ds1, ds2, dnu1, dnu2;  // physical (after the sign flip)
};

__device__ __forceinline__ Dir direction(double beta, double z, double s1, double s2, double y1,
                                         double y2, double nu1, double nu2, double g1, double g2,
                                         double mu, double db, double dz) {
  Dir d;
  const double r3 = sub(y1, dvd(mu, s1));
  const double r4 = sub(y2, dvd(mu, s2));
  const double r5 = sub(add(z, beta), s1);
  const double r6 = sub(sub(z, beta), s2);
  d.dy1 = sub(mul(-g1, add(add(db, dz), r5)), r3);
  d.dy2 = sub(mul(g2, sub(sub(db, dz), r6)), r4);
  d.ds1c = dvd(add(r3, d.dy1), g1);
  d.ds2c = dvd(add(r4, d.dy2), g2);
  d.ds1 = -d.ds1c;
  d.ds2 = -d.ds2c;
  d.dnu1 = sub(dvd(sub(mu, mul(s1, nu1)), s1), mul(g1, d.ds1));
  d.dnu2 = sub(dvd(sub(mu, mul(s2, nu2)), s2), mul(g2, d.ds2));
  return d;
}

#define LOAD_STATE(i)                                                                   \
  const double beta = st.beta[i], z = st.z[i], s1 = st.s1[i], s2 = st.s2[i];              \
  const double y1 = st.y1[i], y2 = st.y2[i], nu1 = st.nu1[i], nu2 = st.nu2[i];

__global__ void k_recover(int64_t n, const double* __restrict__ sig1, const double* __restrict__ sig2,
                          const double* __restrict__ r3p, const double* __restrict__ r4p,
                          const double* __restrict__ r5p, const double* __restrict__ r6p,
                          const double* __restrict__ db, const double* __restrict__ dz, double* ds1,
                          double* ds2, double* dy1, double* dy2) {
  GRID_LOOP(i, n) {
    const double g1 = sig1[i], g2 = sig2[i], r3 = r3p[i], r4 = r4p[i];
    const double b = db[i], c = dz[i];
    const double y1 = sub(mul(-g1, add(add(b, c), r5p[i])), r3);
    const double y2 = sub(mul(g2, sub(sub(b, c), r6p[i])), r4);
    dy1[i] = y1;
    dy2[i] = y2;
    ds1[i] = dvd(add(r3, y1), g1);
    ds2[i] = dvd(add(r4, y2), g2);
  }
}

__global__ void k_direction(int64_t n, fl_state st, const double* __restrict__ sig1,
                            const double* __restrict__ sig2, double mu, const double* __restrict__ db,
                            const double* __restrict__ dz, double* ds1, double* ds2, double* dy1,
                            double* dy2, double* dnu1, double* dnu2) {
  GRID_LOOP(i, n) {
    LOAD_STATE(i)
    const Dir d = direction(beta, z, s1, s2, y1, y2, nu1, nu2, sig1[i], sig2[i], mu, db[i], dz[i]);
    ds1[i] = d.ds1;
    ds2[i] = d.ds2;
    dy1[i] = d.dy1;
    dy2[i] = d.dy2;
    dnu1[i] = d.dnu1;
    dnu2[i] = d.dnu2;
  }
}

// fraction_to_boundary ratio minima (ipm.py:355-361): min over dv<0 of v/(-dv)
__device__ __forceinline__ void ratio_min(double v, double dv, double& acc) {
  if (dv < 0.0) acc = nanmin(acc, dvd(v, -dv));
}

__global__ void k_ratios(int64_t n, fl_state st, const double* __restrict__ sig1,
                         const double* __restrict__ sig2, double mu, const double* __restrict__ db,
                         const double* __restrict__ dz, double* __restrict__ partials) {
  __shared__ double red[32];
  double m1 = INFINITY, m2 = INFINITY, m3 = INFINITY, m4 = INFINITY;
  GRID_LOOP(i, n) {
    LOAD_STATE(i)
    const Dir d = direction(beta, z, s1, s2, y1, y2, nu1, nu2, sig1[i], sig2[i], mu, db[i], dz[i]);
    ratio_min(s1, d.ds1, m1);
    ratio_min(s2, d.ds2, m2);
    ratio_min(nu1, d.dnu1, m3);
    ratio_min(nu2, d.dnu2, m4);
  }
  emit(m1, NanMinOp(), red, partials, 0);
  emit(m2, NanMinOp(), red, partials, 1);
  emit(m3, NanMinOp(), red, partials, 2);
  emit(m4, NanMinOp(), red, partials, 3);
}

__device__ __forceinline__ double step(double v, double a, double dv) { return add(v, mul(a, dv)); }

__global__ void k_update(int64_t n, fl_state st, const double* __restrict__ sig1,
                         const double* __restrict__ sig2, double mu, const double* __restrict__ db,
                         const double* __restrict__ dz, double ap, double ad,
                         double* __restrict__ partials, const double* __restrict__ alpha_dev = nullptr) {
  __shared__ double red[32];
  double flag = 0.0;
  // device step lengths (k_step_alpha): [alpha_p, alpha_d, skip]
  const bool skip = alpha_dev && alpha_dev[2] != 0.0;
  if (alpha_dev) {
    ap = alpha_dev[0];
    ad = alpha_dev[1];
  }
  if (!skip) GRID_LOOP(i, n) {
    LOAD_STATE(i)
    const double b = db[i], c = dz[i];
    const Dir d = direction(beta, z, s1, s2, y1, y2, nu1, nu2, sig1[i], sig2[i], mu, b, c);
    const double n1 = step(s1, ap, d.ds1), n2 = step(s2, ap, d.ds2);
    const double n3 = step(nu1, ad, d.dnu1), n4 = step(nu2, ad, d.dnu2);
    st.beta[i] = step(beta, ap, b);
    st.z[i] = step(z, ap, c);
    st.s1[i] = n1;
    st.s2[i] = n2;
    st.y1[i] = step(y1, ad, d.dy1);
    st.y2[i] = step(y2, ad, d.dy2);
    st.nu1[i] = n3;
    st.nu2[i] = n4;
    if (n1 <= 0.0 || n2 <= 0.0 || n3 <= 0.0 || n4 <= 0.0) flag = 1.0;
  }
  emit(flag, MaxOp(), red, partials, 0);
}

// Step lengths on the device from the four ratio minima (ipm.py:355-361):
// the same IEEE operations as ipm._alpha_from_ratio and Python's min() on the
// host (min(a, b) keeps a unless b < a).  skip = 1 when the PCG verdict is not
// "converged" or the step collapsed (< 1e-12): the gated update then leaves
// the state untouched and the host raises after its one sync.
__device__ __forceinline__ double alpha_of(double ratio, double tau) {
  if (ratio == INFINITY) return 1.0;
  const double a = tau * ratio;
  return a < 1.0 ? a : 1.0;
}
__device__ __forceinline__ double pymin(double a, double b) { return b < a ? b : a; }

__global__ void k_step_alpha(const double* __restrict__ minima, const int* __restrict__ pcg_status,
                             double tau, double* __restrict__ alpha) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double ap = pymin(alpha_of(minima[0], tau), alpha_of(minima[1], tau));
  const double ad = pymin(alpha_of(minima[2], tau), alpha_of(minima[3], tau));
  alpha[0] = ap;
  alpha[1] = ad;
  alpha[2] = (*pcg_status != 1 || pymin(ap, ad) < 1e-12) ? 1.0 : 0.0;
}

__global__ void k_update_explicit(int64_t n, fl_state st, fl_state dir, double ap, double ad,
                                  double* __restrict__ partials) {
  __shared__ double red[32];
  double flag = 0.0;
  GRID_LOOP(i, n) {
    st.beta[i] = step(st.beta[i], ap, dir.beta[i]);
    st.z[i] = step(st.z[i], ap, dir.z[i]);
    const double n1 = step(st.s1[i], ap, dir.s1[i]), n2 = step(st.s2[i], ap, dir.s2[i]);
    st.s1[i] = n1;
    st.s2[i] = n2;
    st.y1[i] = step(st.y1[i], ad, dir.y1[i]);
    st.y2[i] = step(st.y2[i], ad, dir.y2[i]);
    const double n3 = step(st.nu1[i], ad, dir.nu1[i]), n4 = step(st.nu2[i], ad, dir.nu2[i]);
    st.nu1[i] = n3;
    st.nu2[i] = n4;
    if (n1 <= 0.0 || n2 <= 0.0 || n3 <= 0.0 || n4 <= 0.0) flag = 1.0;
  }
  emit(flag, MaxOp(), red, partials, 0);
}

// ---------------- initial state / assessment (ipm.py:214-282) ----------------
__global__ void k_init(int64_t n, fl_state st, double half) {
  GRID_LOOP(i, n) {
    st.beta[i] = 0.0;
    st.z[i] = 1.0;
    st.s1[i] = 1.0;
    st.s2[i] = 1.0;
    st.y1[i] = half;
    st.y2[i] = half;
    st.nu1[i] = half;
    st.nu2[i] = half;
  }
}

__global__ void k_assess(int64_t n, fl_state st, const double* __restrict__ g, double lam, double mu,
                         double* __restrict__ partials) {
  __shared__ double red[32];
  double a_stat = 0.0, a_dual = 0.0, a_gap = 0.0, a_pr = 0.0;
  double a_cmax = -INFINITY, a_cmin = INFINITY, a_d1 = 0.0, a_d2 = 0.0, a_bar = 0.0;
  GRID_LOOP(i, n) {
    LOAD_STATE(i)
    const double stat = fabs(sub(add(g[i], y1), y2));
    const double dual = fabs(sub(sub(lam, y1), y2));
    const double r2 = fabs(sub(add(y1, y2), lam));
    const double gap1 = fabs(sub(y1, nu1)), gap2 = fabs(sub(y2, nu2));
    const double pr1 = fabs(sub(add(z, beta), s1)), pr2 = fabs(sub(sub(z, beta), s2));
    const double p1 = mul(s1, nu1), p2 = mul(s2, nu2);
    a_stat = nanmax(a_stat, stat);
    a_dual = nanmax(a_dual, dual);
    a_gap = nanmax(a_gap, nanmax(gap1, gap2));
    a_pr = nanmax(a_pr, nanmax(pr1, pr2));
    a_cmax = nanmax(a_cmax, nanmax(p1, p2));
    a_cmin = nanmin(a_cmin, nanmin(p1, p2));
    a_d1 += mul(nu1, s1);
    a_d2 += mul(nu2, s2);
    const double c1 = fabs(sub(p1, mu)), c2 = fabs(sub(p2, mu));
    a_bar = nanmax(a_bar, nanmax(nanmax(nanmax(stat, r2), nanmax(pr1, pr2)),
                                 nanmax(nanmax(c1, c2), nanmax(gap1, gap2))));
  }
  emit(a_stat, NanMaxOp(), red, partials, 0);
  emit(a_dual, NanMaxOp(), red, partials, 1);
  emit(a_gap, NanMaxOp(), red, partials, 2);
  emit(a_pr, NanMaxOp(), red, partials, 3);
  emit(a_cmax, NanMaxOp(), red, partials, 4);
  emit(a_cmin, NanMinOp(), red, partials, 5);
  emit(a_d1, SumOp(), red, partials, 6);
  emit(a_d2, SumOp(), red, partials, 7);
  emit(a_bar, NanMaxOp(), red, partials, 8);
}

// lasso objective pieces (ipm.py:209-211): sum over observed (b - x)^2, sum |beta|
__global__ void k_objective(int64_t n, const uint32_t* __restrict__ bits, const double* __restrict__ bhat,
                            const double* __restrict__ x, const double* __restrict__ beta,
                            double* __restrict__ partials) {
  __shared__ double red[32];
  double ss = 0.0, l1 = 0.0;
  GRID_LOOP(i, n) {
    const bool miss = (bits[i >> 5] >> (i & 31)) & 1u;
    if (!miss) {
      const double r = sub(bhat[i], x[i]);
      ss += mul(r, r);
    }
    l1 += fabs(beta[i]);
  }
  emit(ss, SumOp(), red, partials, 0);
  emit(l1, SumOp(), red, partials, 1);
}

// ---------------- generic vector primitives ----------------
__global__ void k_dot(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ partials) {
  __shared__ double red[32];
  double s = 0.0;
  GRID_LOOP(i, n) s += mul(a[i], b[i]);
  emit(s, SumOp(), red, partials, 0);
}

__global__ void k_maxabs(int64_t n, const double* __restrict__ a, double* __restrict__ partials) {
  __shared__ double red[32];
  double s = 0.0;
  GRID_LOOP(i, n) s = nanmax(s, fabs(a[i]));
  emit(s, NanMaxOp(), red, partials, 0);
}

__global__ void k_min(int64_t n, const double* __restrict__ a, double* __restrict__ partials) {
  __shared__ double red[32];
  double s = INFINITY;
  GRID_LOOP(i, n) s = nanmin(s, a[i]);
  emit(s, NanMinOp(), red, partials, 0);
}

__global__ void k_ftb(int64_t n, const double* __restrict__ v, const double* __restrict__ dv,
                      double* __restrict__ partials) {
  __shared__ double red[32];
  double s = INFINITY;
  GRID_LOOP(i, n) ratio_min(v[i], dv[i], s);
  emit(s, NanMinOp(), red, partials, 0);
}

// np.sign(x) * np.maximum(np.abs(x) - t, 0.0) (diagnostics.py:325-328) with
// NumPy's conventions: sign(+-0) = +0, sign(NaN) = NaN, maximum(m, 0) = m only
// when m > 0 or m is NaN (so -0.0 becomes +0.0).
__device__ __forceinline__ double soft(double x, double t) {
  const double sg = x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : (x == x ? 0.0 : x));
  const double m = sub(fabs(x), t);
  return mul(sg, (m > 0.0 || isnan(m)) ? m : 0.0);
}

__global__ void k_soft(int64_t n, const double* __restrict__ x, double t, double* __restrict__ out) {
  GRID_LOOP(i, n) out[i] = soft(x[i], t);
}

// One ISTA iteration (diagnostics.py:352-357) after the gram: grad = G beta - xi,
// next = soft(beta - grad, lam), step = max |next - beta| (NaN-propagating).
__global__ void k_ista(int64_t n, const double* __restrict__ beta, const double* __restrict__ gb,
                       const double* __restrict__ xi, double lam, double* __restrict__ next,
                       double* __restrict__ partials) {
  __shared__ double red[32];
  double s = 0.0;
  GRID_LOOP(i, n) {
    const double b = beta[i];
    const double nx = soft(sub(b, sub(gb[i], xi[i])), lam);
    next[i] = nx;
    s = nanmax(s, fabs(sub(nx, b)));
  }
  emit(s, NanMaxOp(), red, partials, 0);
}

__global__ void k_axpy(int64_t n, double alpha, const double* __restrict__ x, double* __restrict__ y) {
  GRID_LOOP(i, n) y[i] = add(y[i], mul(alpha, x[i]));
}

__global__ void k_xpby(int64_t n, const double* __restrict__ x, double beta, double* __restrict__ y) {
  GRID_LOOP(i, n) y[i] = add(x[i], mul(beta, y[i]));
}

// ---------------- PCG on the condensed system (pcg.py:84-127) ----------------
// 2n vectors are [beta-block (n); z-block (n)].
// KKT epilogue (newton_system.py:150-151) on the gram output g, in place:
// top = (g + L1 pb) + L2 pz, bottom = L2 pb + L1 pz, partial d.Kd.  16-byte
// accesses (n is even for every grid).
__global__ void k_kkt_epilogue(int64_t n2, double2* __restrict__ g, const double2* __restrict__ pb,
                               const double2* __restrict__ pz, const double2* __restrict__ s1,
                               const double2* __restrict__ s2, double2* __restrict__ bot,
                               double* __restrict__ partials) {
  __shared__ double red[32];
  double acc = 0.0;
  GRID_LOOP(i, n2) {
    const double2 gv = g[i], b = pb[i], z = pz[i], a1 = s1[i], a2 = s2[i];
    double2 t, u;
    double l1 = add(a1.x, a2.x), l2 = sub(a1.x, a2.x);
    t.x = add(add(gv.x, mul(l1, b.x)), mul(l2, z.x));
    u.x = add(mul(l2, b.x), mul(l1, z.x));
    l1 = add(a1.y, a2.y);
    l2 = sub(a1.y, a2.y);
    t.y = add(add(gv.y, mul(l1, b.y)), mul(l2, z.y));
    u.y = add(mul(l2, b.y), mul(l1, z.y));
    g[i] = t;
    if (bot) bot[i] = u;
    acc += mul(b.x, t.x) + mul(z.x, u.x) + mul(b.y, t.y) + mul(z.y, u.y);
  }
  if (partials) emit(acc, SumOp(), red, partials, 0);
}

// ---- restructured PCG (g = G p_beta instead of materialised K p) ----
// d.(K - G)d = pb (L1 pb + L2 pz) + pz (L2 pb + L1 pz): the diagonal part of
// the curvature, accumulated where p is written (init / p-update).
__device__ __forceinline__ double diag_quad(double l1, double l2, double pb, double pz) {
  return pb * (l1 * pb + l2 * pz) + pz * (l2 * pb + l1 * pz);
}

__global__ void k_pcg2_init(int64_t n, const double* __restrict__ g1, const double* __restrict__ g2,
                            const double* __restrict__ rhs, double* __restrict__ x,
                            double* __restrict__ r, double* __restrict__ p, double* __restrict__ partials) {
  __shared__ double red[32];
  double rho = 0.0, dq = 0.0;
  GRID_LOOP(i, n) {
    const double rb = rhs[i], rc = rhs[n + i];
    const Pinv P(g1[i], g2[i]);
    const double zt = P.top(rb, rc), zb = P.bot(rb, rc);
    x[i] = 0.0;
    x[n + i] = 0.0;
    r[i] = rb;
    r[n + i] = rc;
    p[i] = zt;
    p[n + i] = zb;
    rho += mul(rb, zt) + mul(rc, zb);
    dq += diag_quad(P.l1, P.l2, zt, zb);
  }
  emit(rho, SumOp(), red, partials, 0);
  emit(dq, SumOp(), red, partials, 1);
}

// One pass per IPM iteration for everything before the first PCG matvec
// (ipm.py:303-327): barrier diagonals with the interior check
// (newton_system.py:72-91), the condensed RHS (:113-145) and the PCG start
// x = 0, r = rhs, p = P^{-1} r with the rho / diagonal-curvature partials --
// the same formulas and accumulation order as k_diagonals, k_newton_rhs and
// k_pcg2_init, so the results are bitwise those of the three-kernel path.
// Reads 9 n-vectors, writes 8 (136 B/voxel instead of 216).
__global__ void k_newton_setup(int64_t n, fl_state st, const double* __restrict__ g, double lam, double mu,
                               double* __restrict__ sig1, double* __restrict__ sig2, double* __restrict__ x,
                               double* __restrict__ r, double* __restrict__ p, double* __restrict__ partials) {
  __shared__ double red[32];
  double rho = 0.0, dq = 0.0, flag = 0.0;
  GRID_LOOP(i, n) {
    const double beta = st.beta[i], z = st.z[i], s1 = st.s1[i], s2 = st.s2[i];
    const double y1 = st.y1[i], y2 = st.y2[i], nu1 = st.nu1[i], nu2 = st.nu2[i];
    if (bad(s1) || bad(s2) || bad(nu1) || bad(nu2)) flag = 1.0;
    const double g1 = dvd(nu1, s1), g2 = dvd(nu2, s2);
    sig1[i] = g1;
    sig2[i] = g2;
    const double r1 = sub(add(g[i], y1), y2);
    const double r2 = sub(add(y1, y2), lam);
    const double r3 = sub(y1, dvd(mu, s1));
    const double r4 = sub(y2, dvd(mu, s2));
    const double r5 = sub(add(z, beta), s1);
    const double r6 = sub(sub(z, beta), s2);
    const double rb = add(sub(add(sub(r1, r3), r4), mul(g1, r5)), mul(g2, r6));
    const double rc = sub(sub(sub(sub(r2, r3), r4), mul(g1, r5)), mul(g2, r6));
    const Pinv P(g1, g2);
    const double zt = P.top(rb, rc), zb = P.bot(rb, rc);
    x[i] = 0.0;
    x[n + i] = 0.0;
    r[i] = rb;
    r[n + i] = rc;
    p[i] = zt;
    p[n + i] = zb;
    rho += mul(rb, zt) + mul(rc, zb);
    dq += diag_quad(P.l1, P.l2, zt, zb);
  }
  emit(rho, SumOp(), red, partials, 0);
  emit(dq, SumOp(), red, partials, 1);
  emit(flag, MaxOp(), red, partials, 2);
}

// x += alpha p; r -= alpha K p with K p formed in registers from g = G p_beta
// exactly as apply_kkt (newton_system.py:150-151); z = P^{-1} r; rho partials.
// 16-byte accesses: each thread handles voxels (2i, 2i+1) of both blocks.
struct KUpd {
  __device__ __forceinline__ static void one(double a1, double a2, double alpha, double g, double pt,
                                             double pb, double& xt, double& xb, double& rt, double& rb,
                                             double& rho) {
    const double l1 = add(a1, a2), l2 = sub(a1, a2);
    const double kt = add(add(g, mul(l1, pt)), mul(l2, pb));
    const double kb = add(mul(l2, pt), mul(l1, pb));
    xt = add(xt, mul(alpha, pt));
    xb = add(xb, mul(alpha, pb));
    rt = sub(rt, mul(alpha, kt));
    rb = sub(rb, mul(alpha, kb));
    const Pinv P(a1, a2);
    rho += mul(rt, P.top(rt, rb)) + mul(rb, P.bot(rt, rb));
  }
};

__global__ void k_pcg2_update(int64_t n, const double* __restrict__ g1, const double* __restrict__ g2,
                              const double* __restrict__ rho_p, const double* __restrict__ curv_g,
                              const double* __restrict__ curv_d, double* __restrict__ x,
                              double* __restrict__ r, const double* __restrict__ p,
                              const double* __restrict__ gp, double* __restrict__ partials) {
  __shared__ double red[32];
  const double alpha = dvd(*rho_p, add(*curv_g, *curv_d));
  double rho = 0.0;
  const int64_t n2 = n >> 1;
  const double2* G1 = reinterpret_cast<const double2*>(g1);
  const double2* G2 = reinterpret_cast<const double2*>(g2);
  const double2* PT = reinterpret_cast<const double2*>(p);
  const double2* PB = reinterpret_cast<const double2*>(p + n);
  const double2* GP = reinterpret_cast<const double2*>(gp);
  double2* XT = reinterpret_cast<double2*>(x);
  double2* XB = reinterpret_cast<double2*>(x + n);
  double2* RT = reinterpret_cast<double2*>(r);
  double2* RB = reinterpret_cast<double2*>(r + n);
  GRID_LOOP(i, n2) {
    const double2 a1 = G1[i], a2 = G2[i], pt = PT[i], pb = PB[i], g = GP[i];
    double2 xt = XT[i], xb = XB[i], rt = RT[i], rb = RB[i];
    KUpd::one(a1.x, a2.x, alpha, g.x, pt.x, pb.x, xt.x, xb.x, rt.x, rb.x, rho);
    KUpd::one(a1.y, a2.y, alpha, g.y, pt.y, pb.y, xt.y, xb.y, rt.y, rb.y, rho);
    XT[i] = xt;
    XB[i] = xb;
    RT[i] = rt;
    RB[i] = rb;
  }
  emit(rho, SumOp(), red, partials, 0);
}

__global__ void k_pcg2_pupdate(int64_t n, const double* __restrict__ g1, const double* __restrict__ g2,
                               const double* __restrict__ r, double beta, double* __restrict__ p,
                               double* __restrict__ partials, const double* __restrict__ beta_dev,
                               const int* __restrict__ done) {
  __shared__ double red[32];
  if (done && *done) return;
  if (beta_dev) beta = *beta_dev;
  double dq = 0.0;
  const int64_t n2 = n >> 1;
  const double2* G1 = reinterpret_cast<const double2*>(g1);
  const double2* G2 = reinterpret_cast<const double2*>(g2);
  const double2* RT = reinterpret_cast<const double2*>(r);
  const double2* RB = reinterpret_cast<const double2*>(r + n);
  double2* PT = reinterpret_cast<double2*>(p);
  double2* PB = reinterpret_cast<double2*>(p + n);
  GRID_LOOP(i, n2) {
    const double2 a1 = G1[i], a2 = G2[i], rt = RT[i], rb = RB[i];
    double2 pt = PT[i], pb = PB[i];
    {
      const Pinv P(a1.x, a2.x);
      pt.x = add(P.top(rt.x, rb.x), mul(beta, pt.x));
      pb.x = add(P.bot(rt.x, rb.x), mul(beta, pb.x));
      dq += diag_quad(P.l1, P.l2, pt.x, pb.x);
    }
    {
      const Pinv P(a1.y, a2.y);
      pt.y = add(P.top(rt.y, rb.y), mul(beta, pt.y));
      pb.y = add(P.bot(rt.y, rb.y), mul(beta, pb.y));
      dq += diag_quad(P.l1, P.l2, pt.y, pb.y);
    }
    PT[i] = pt;
    PB[i] = pb;
  }
  emit(dq, SumOp(), red, partials, 0);
}

// alpha by value (host-driven sharded loop) or from device memory
// (alpha_dev != nullptr: the device-scalar sharded loop, fl_pcg_step_alpha)
__global__ void k_pcg2_update_a(int64_t n, const double* __restrict__ g1, const double* __restrict__ g2,
                                double alpha_v, const double* __restrict__ alpha_dev, double* __restrict__ x,
                                double* __restrict__ r, const double* __restrict__ p,
                                const double* __restrict__ gp, double* __restrict__ partials) {
  __shared__ double red[32];
  const double alpha = alpha_dev ? *alpha_dev : alpha_v;
  double rho = 0.0;
  GRID_LOOP(i, n) {
    const double pt = p[i], pb = p[n + i];
    const double a1 = g1[i], a2 = g2[i];
    const double l1 = add(a1, a2), l2 = sub(a1, a2);
    const double kt = add(add(gp[i], mul(l1, pt)), mul(l2, pb));
    const double kb = add(mul(l2, pt), mul(l1, pb));
    x[i] = add(x[i], mul(alpha, pt));
    x[n + i] = add(x[n + i], mul(alpha, pb));
    const double rt = sub(r[i], mul(alpha, kt));
    const double rb = sub(r[n + i], mul(alpha, kb));
    r[i] = rt;
    r[n + i] = rb;
    const Pinv P(a1, a2);
    rho += mul(rt, P.top(rt, rb)) + mul(rb, P.bot(rt, rb));
  }
  emit(rho, SumOp(), red, partials, 0);
}

__global__ void k_step_alpha_dev(const double* __restrict__ red2, const double* __restrict__ rho,
                                 double* __restrict__ out) {
  if (threadIdx.x == 0) {
    const double curv = add(red2[0], red2[1]);
    out[0] = curv;
    out[1] = dvd(rho[0], curv);
  }
}

__global__ void k_objective_terms(int64_t n, const uint32_t* __restrict__ bits, const double* __restrict__ bhat,
                                  const double* __restrict__ x, int64_t nb, const double* __restrict__ beta,
                                  double* __restrict__ partials) {
  __shared__ double red[32];
  double ss = 0.0, l1 = 0.0;
  GRID_LOOP(i, n) {
    if (!((bits[i >> 5] >> (i & 31)) & 1u)) {
      const double r = sub(bhat[i], x[i]);
      ss += mul(r, r);
    }
  }
  if (beta) GRID_LOOP(i, nb) l1 += fabs(beta[i]);
  emit(ss, SumOp(), red, partials, 0);
  emit(l1, SumOp(), red, partials, 1);
}

// Reduce ``nk`` partial rows and fetch them to the host.
int reduce_fetch(Scratch* sc, int grid, int nk, const int* kinds, double* out, cudaStream_t s) {
  FL_TRY(finish_reduce(sc->partials, grid, nk, kinds, sc->result, s));
  FL_TRY(fetch_results(sc, nk, s));
  for (int k = 0; k < nk; ++k) out[k] = sc->host[k];
  return FL_OK;
}

}  // namespace

// ---- internal entry points used by the PCG driver ----
int kkt_epilogue(int64_t n, double* g, const double* pb, const double* pz, const double* sig1,
                 const double* sig2, double* bottom, double* partials, int* nblocks, cudaStream_t s) {
  const int64_t n2 = n / 2;
  const int grid = grid_for(n2, T, 148 * 16);
  k_kkt_epilogue<<<grid, T, 0, s>>>(n2, reinterpret_cast<double2*>(g), reinterpret_cast<const double2*>(pb),
                                    reinterpret_cast<const double2*>(pz), reinterpret_cast<const double2*>(sig1),
                                    reinterpret_cast<const double2*>(sig2), reinterpret_cast<double2*>(bottom),
                                    partials);
  FL_LAUNCH_CHECK();
  if (nblocks) *nblocks = grid;
  return FL_OK;
}

int pcg2_init(int64_t n, const double* sig1, const double* sig2, const double* rhs, double* x, double* r,
              double* p, double* partials, int* nblocks, cudaStream_t s) {
  const int grid = grid_for(n, T);
  k_pcg2_init<<<grid, T, 0, s>>>(n, sig1, sig2, rhs, x, r, p, partials);
  FL_LAUNCH_CHECK();
  *nblocks = grid;
  return FL_OK;
}

int newton_setup(int64_t n, const fl_state* st, const double* g, double lam, double mu, double* sig1,
                 double* sig2, double* x, double* r, double* p, double* partials, int* nblocks, cudaStream_t s) {
  const int grid = grid_for(n, T);
  k_newton_setup<<<grid, T, 0, s>>>(n, *st, g, lam, mu, sig1, sig2, x, r, p, partials);
  FL_LAUNCH_CHECK();
  *nblocks = grid;
  return FL_OK;
}

int pcg2_update(int64_t n, const double* sig1, const double* sig2, const double* rho, const double* curv_g,
                const double* curv_d, double* x, double* r, const double* p, const double* gp,
                double* partials, int* nblocks, cudaStream_t s) {
  if (n % 2) return fail(FL_E_SHAPE, "PCG update needs an even length (16-byte accesses)");
  const int grid = grid_for(n, T);
  k_pcg2_update<<<grid, T, 0, s>>>(n, sig1, sig2, rho, curv_g, curv_d, x, r, p, gp, partials);
  FL_LAUNCH_CHECK();
  *nblocks = grid;
  return FL_OK;
}

int pcg2_pupdate(int64_t n, const double* sig1, const double* sig2, const double* r, double beta, double* p,
                 double* partials, int* nblocks, cudaStream_t s, const double* beta_dev, const int* done) {
  if (n % 2) return fail(FL_E_SHAPE, "PCG p-update needs an even length (16-byte accesses)");
  const int grid = grid_for(n, T);
  k_pcg2_pupdate<<<grid, T, 0, s>>>(n, sig1, sig2, r, beta, p, partials, beta_dev, done);
  FL_LAUNCH_CHECK();
  *nblocks = grid;
  return FL_OK;
}

int dot_partials(int64_t n, const double* a, const double* b, double* partials, int* nblocks, cudaStream_t s) {
  const int grid = grid_for(n, T);
  k_dot<<<grid, T, 0, s>>>(n, a, b, partials);
  FL_LAUNCH_CHECK();
  *nblocks = grid;
  return FL_OK;
}

// Back half of the IPM step with no host sync (ipm.py:364-394): ratio minima
// -> dev[0..3], step lengths -> dev[4..6] (gated on *pcg_status), the state
// update, interior flag -> dev[7].
int ipm_step_device(int64_t n, const fl_state* st, const double* sigma1, const double* sigma2, double mu,
                    double tau, const double* d_beta, const double* d_z, const int* pcg_status, double* dev,
                    cudaStream_t s) {
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_ratios<<<grid, T, 0, s>>>(n, *st, sigma1, sigma2, mu, d_beta, d_z, sc->partials);
  FL_LAUNCH_CHECK();
  const int kinds[4] = {RED_MIN, RED_MIN, RED_MIN, RED_MIN};
  FL_TRY(finish_reduce(sc->partials, grid, 4, kinds, dev, s));
  k_step_alpha<<<1, 32, 0, s>>>(dev, pcg_status, tau, dev + 4);
  FL_LAUNCH_CHECK();
  k_update<<<grid, T, 0, s>>>(n, *st, sigma1, sigma2, mu, d_beta, d_z, 0.0, 0.0, sc->partials, dev + 4);
  FL_LAUNCH_CHECK();
  const int kind = RED_MAX;
  return finish_reduce(sc->partials, grid, 1, &kind, dev + 7, s);
}

}  // namespace fl

using namespace fl;

extern "C" {

// offsets[w] = observed samples before word w (exclusive scan of the
// per-word observed counts already in `offsets`); *n_observed = total.
static int mask_offsets(int64_t nw, int64_t* offsets, int64_t* n_observed, cudaStream_t s) {
  int64_t last_count = 0;
  FL_CUDA(cudaMemcpyAsync(&last_count, offsets + nw - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  size_t tmp_bytes = 0;
  FL_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, offsets, offsets, (int)nw, s));
  void* tmp = nullptr;
  FL_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));
  cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, offsets, offsets, (int)nw, s);
  cudaFreeAsync(tmp, s);
  FL_CUDA(e);
  int64_t last_off = 0;
  FL_CUDA(cudaMemcpyAsync(&last_off, offsets + nw - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FL_CUDA(cudaStreamSynchronize(s));
  if (n_observed) *n_observed = last_off + last_count;
  return FL_OK;
}

int fl_mask_build(int64_t n, const uint8_t* flags, uint32_t* bits, int64_t* offsets,
                  int64_t* n_observed, fl_stream_t stream) {
  if (n <= 0 || !flags || !bits || !offsets) return fail(FL_E_VALUE, "bad mask arguments");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nw = (n + 31) >> 5;
  k_mask_bits<<<grid_for(nw, T, 1 << 16), T, 0, s>>>(n, flags, bits, offsets);
  FL_LAUNCH_CHECK();
  return mask_offsets(nw, offsets, n_observed, s);
}

int fl_mask_bragg(int ndim, const int64_t* dims, int64_t spacing, double radius, uint32_t* bits,
                  int64_t* offsets, int64_t* n_observed, fl_stream_t stream) {
  if (ndim < 1 || ndim > 3 || !dims || spacing < 1 || !bits || !offsets) return fail(FL_E_VALUE, "bad mask arguments");
  int64_t n = 1;
  for (int a = 0; a < ndim; ++a) {
    if (dims[a] < 1) return fail(FL_E_SHAPE, "bad grid extent");
    n *= dims[a];
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nw = (n + 31) >> 5;
  const int64_t d2 = dims[ndim - 1], d1 = ndim >= 2 ? dims[ndim - 2] : 1;
  k_bragg_bits<<<grid_for(nw, T, 1 << 16), T, 0, s>>>(n, ndim, d1, d2, spacing, radius * radius, bits, offsets);
  FL_LAUNCH_CHECK();
  return mask_offsets(nw, offsets, n_observed, s);
}

int fl_noisy_embed(const int64_t* ext, const int64_t* off, const int64_t* stride, uint64_t seed, double sigma,
                   const uint32_t* miss_bits, double* x, fl_stream_t stream) {
  if (!ext || !off || !stride || !miss_bits || !x) return fail(FL_E_VALUE, "null argument");
  if (ext[0] < 0 || ext[1] < 1 || ext[2] < 1) return fail(FL_E_SHAPE, "bad local box");
  const int64_t nl = ext[0] * ext[1] * ext[2];
  if (nl == 0) return FL_OK;
  k_noisy_embed<<<grid_for(nl, T, 1 << 16), T, 0, (cudaStream_t)stream>>>(
      nl, ext[1], ext[2], off[0], off[1], off[2], stride[0], stride[1], stride[2], seed, sigma, miss_bits, x);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fl_embed(int64_t n, const uint32_t* bits, const int64_t* off, const double* obs, double* full,
             fl_stream_t stream) {
  if (!bits || !off || !full || (!obs && n)) return fail(FL_E_VALUE, "null argument");
  k_embed<<<grid_for(n, T, 1 << 16), T, 0, (cudaStream_t)stream>>>(n, bits, off, obs, full);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fl_gather_observed(int64_t n, const uint32_t* bits, const int64_t* off, const double* full,
                       double* obs, fl_stream_t stream) {
  if (!bits || !off || !full || !obs) return fail(FL_E_VALUE, "null argument");
  k_gather<<<grid_for(n, T, 1 << 16), T, 0, (cudaStream_t)stream>>>(n, bits, off, full, obs);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fl_barrier_diagonals(int64_t n, const double* s1, const double* s2, const double* nu1,
                         const double* nu2, double* sigma1, double* sigma2, double* lambda1,
                         double* lambda2, double* dvec, double* bvec, fl_stream_t stream) {
  if (n <= 0) return fail(FL_E_INTERIOR, "s1 must be strictly positive and finite");
  if (!s1 || !s2 || !nu1 || !nu2 || !sigma1 || !sigma2) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_diagonals<<<grid, T, 0, s>>>(n, s1, s2, nu1, nu2, sigma1, sigma2, lambda1, lambda2, dvec, bvec,
                                 sc->partials);
  FL_LAUNCH_CHECK();
  const int kind = RED_MAX;
  double flag = 0.0;
  FL_TRY(reduce_fetch(sc, grid, 1, &kind, &flag, s));
  if (flag != 0.0) return fail(FL_E_INTERIOR, "slacks and multipliers must be strictly positive and finite");
  return FL_OK;
}

int fl_precond_apply(int64_t n, const double* sigma1, const double* sigma2, const double* r_beta,
                     const double* r_c, double* top, double* bottom, fl_stream_t stream) {
  if (!sigma1 || !sigma2 || !r_beta || !r_c || !top || !bottom) return fail(FL_E_VALUE, "null argument");
  k_precond<<<grid_for(n, T), T, 0, (cudaStream_t)stream>>>(n, sigma1, sigma2, r_beta, r_c, top, bottom);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fl_newton_rhs(int64_t n, const fl_state* st, const double* g, const double* sigma1,
                  const double* sigma2, double lam, double mu, double* r1, double* r2, double* r3,
                  double* r4, double* r5, double* r6, double* r_beta, double* r_c,
                  fl_stream_t stream) {
  if (!st || !g || !sigma1 || !sigma2 || !r_beta || !r_c) return fail(FL_E_VALUE, "null argument");
  k_newton_rhs<<<grid_for(n, T), T, 0, (cudaStream_t)stream>>>(n, *st, g, sigma1, sigma2, lam, mu, r1,
                                                                r2, r3, r4, r5, r6, r_beta, r_c);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fl_recover_eliminated(int64_t n, const double* sigma1, const double* sigma2, const double* r3,
                          const double* r4, const double* r5, const double* r6, const double* d_beta,
                          const double* d_z, double* d_s1, double* d_s2, double* d_y1, double* d_y2,
                          fl_stream_t stream) {
  if (!sigma1 || !sigma2 || !r3 || !r4 || !r5 || !r6 || !d_beta || !d_z || !d_s1 || !d_s2 || !d_y1 ||
      !d_y2)
    return fail(FL_E_VALUE, "null argument");
  k_recover<<<grid_for(n, T), T, 0, (cudaStream_t)stream>>>(n, sigma1, sigma2, r3, r4, r5, r6, d_beta,
                                                             d_z, d_s1, d_s2, d_y1, d_y2);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fl_ipm_init(int64_t n, const fl_state* st, double lam, fl_stream_t stream) {
  if (!st) return fail(FL_E_VALUE, "null argument");
  if (!(lam > 0)) return fail(FL_E_VALUE, "penalty must be positive");
  k_init<<<grid_for(n, T), T, 0, (cudaStream_t)stream>>>(n, *st, 0.5 * lam);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fl_ipm_assess(int64_t n, const fl_state* st, const double* g, double lam, double mu,
                  fl_assess* out, fl_stream_t stream) {
  if (!st || !g || !out) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_assess<<<grid, T, 0, s>>>(n, *st, g, lam, mu, sc->partials);
  FL_LAUNCH_CHECK();
  const int kinds[9] = {RED_MAX, RED_MAX, RED_MAX, RED_MAX, RED_MAX, RED_MIN, RED_SUM, RED_SUM, RED_MAX};
  double v[9];
  FL_TRY(reduce_fetch(sc, grid, 9, kinds, v, s));
  out->stationarity = v[0];
  out->dual_equality = v[1];
  out->multiplier_gap = v[2];
  out->primal = v[3];
  out->complementarity = v[4];
  out->min_product = v[5];
  out->dot_nu_s1 = v[6];
  out->dot_nu_s2 = v[7];
  out->barrier_residual = v[8];
  return FL_OK;
}

int fl_ipm_ratios(int64_t n, const fl_state* st, const double* sigma1, const double* sigma2,
                  double mu, const double* d_beta, const double* d_z, double* ratios,
                  fl_stream_t stream) {
  if (!st || !sigma1 || !sigma2 || !d_beta || !d_z || !ratios) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_ratios<<<grid, T, 0, s>>>(n, *st, sigma1, sigma2, mu, d_beta, d_z, sc->partials);
  FL_LAUNCH_CHECK();
  const int kinds[4] = {RED_MIN, RED_MIN, RED_MIN, RED_MIN};
  return reduce_fetch(sc, grid, 4, kinds, ratios, s);
}

int fl_ipm_direction(int64_t n, const fl_state* st, const double* sigma1, const double* sigma2,
                     double mu, const double* d_beta, const double* d_z, double* d_s1, double* d_s2,
                     double* d_y1, double* d_y2, double* d_nu1, double* d_nu2, fl_stream_t stream) {
  if (!st || !sigma1 || !sigma2 || !d_beta || !d_z || !d_s1 || !d_s2 || !d_y1 || !d_y2 || !d_nu1 || !d_nu2)
    return fail(FL_E_VALUE, "null argument");
  k_direction<<<grid_for(n, T), T, 0, (cudaStream_t)stream>>>(n, *st, sigma1, sigma2, mu, d_beta, d_z,
                                                               d_s1, d_s2, d_y1, d_y2, d_nu1, d_nu2);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fl_ipm_update(int64_t n, const fl_state* st, const double* sigma1, const double* sigma2,
                  double mu, const double* d_beta, const double* d_z, double alpha_p,
                  double alpha_d, fl_stream_t stream) {
  if (!st || !sigma1 || !sigma2 || !d_beta || !d_z) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_update<<<grid, T, 0, s>>>(n, *st, sigma1, sigma2, mu, d_beta, d_z, alpha_p, alpha_d, sc->partials);
  FL_LAUNCH_CHECK();
  const int kind = RED_MAX;
  double flag = 0.0;
  FL_TRY(reduce_fetch(sc, grid, 1, &kind, &flag, s));
  if (flag != 0.0) return fail(FL_E_STALLED, "slack or multiplier left the strict interior");
  return FL_OK;
}

int fl_ipm_update_explicit(int64_t n, const fl_state* st, const fl_state* dir, double alpha_p,
                           double alpha_d, fl_stream_t stream) {
  if (!st || !dir) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_update_explicit<<<grid, T, 0, s>>>(n, *st, *dir, alpha_p, alpha_d, sc->partials);
  FL_LAUNCH_CHECK();
  const int kind = RED_MAX;
  double flag = 0.0;
  FL_TRY(reduce_fetch(sc, grid, 1, &kind, &flag, s));
  if (flag != 0.0) return fail(FL_E_STALLED, "slack or multiplier left the strict interior");
  return FL_OK;
}

int fl_lasso_objective(fl_plan_t p, const uint32_t* bits, const double* bhat, const double* beta,
                       double lam, double* work, double* out, fl_stream_t stream) {
  if (!p || !bits || !bhat || !beta || !work || !out) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  FL_TRY(op_synthesize(p, beta, work, s));
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(p->n, T);
  k_objective<<<grid, T, 0, s>>>(p->n, bits, bhat, work, beta, sc->partials);
  FL_LAUNCH_CHECK();
  const int kinds[2] = {RED_SUM, RED_SUM};
  double v[2];
  FL_TRY(reduce_fetch(sc, grid, 2, kinds, v, s));
  *out = 0.5 * v[0] + lam * v[1];
  return FL_OK;
}

int fl_dot(int64_t n, const double* a, const double* b, double* out, fl_stream_t stream) {
  if (!a || !b || !out) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_dot<<<grid, T, 0, s>>>(n, a, b, sc->partials);
  FL_LAUNCH_CHECK();
  const int kind = RED_SUM;
  return reduce_fetch(sc, grid, 1, &kind, out, s);
}

int fl_max_abs(int64_t n, const double* a, double* out, fl_stream_t stream) {
  if (!a || !out) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_maxabs<<<grid, T, 0, s>>>(n, a, sc->partials);
  FL_LAUNCH_CHECK();
  const int kind = RED_MAX;
  return reduce_fetch(sc, grid, 1, &kind, out, s);
}

int fl_min(int64_t n, const double* a, double* out, fl_stream_t stream) {
  if (!a || !out) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_min<<<grid, T, 0, s>>>(n, a, sc->partials);
  FL_LAUNCH_CHECK();
  const int kind = RED_MIN;
  return reduce_fetch(sc, grid, 1, &kind, out, s);
}

int fl_ftb_ratio(int64_t n, const double* v, const double* dv, double* out, fl_stream_t stream) {
  if (!v || !dv || !out) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_ftb<<<grid, T, 0, s>>>(n, v, dv, sc->partials);
  FL_LAUNCH_CHECK();
  const int kind = RED_MIN;
  return reduce_fetch(sc, grid, 1, &kind, out, s);
}

int fl_soft_threshold(int64_t n, const double* x, double t, double* out, fl_stream_t stream) {
  if (n < 0 || (n && (!x || !out))) return fail(FL_E_VALUE, "null argument");
  if (n == 0) return FL_OK;
  k_soft<<<grid_for(n, T), T, 0, (cudaStream_t)stream>>>(n, x, t, out);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fl_ista_step(int64_t n, const double* beta, const double* gram_beta, const double* xi, double lam,
                 double* next, double* step, fl_stream_t stream) {
  if (n <= 0 || !beta || !gram_beta || !xi || !next || !step) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_ista<<<grid, T, 0, s>>>(n, beta, gram_beta, xi, lam, next, sc->partials);
  FL_LAUNCH_CHECK();
  const int kind = RED_MAX;
  return reduce_fetch(sc, grid, 1, &kind, step, s);
}

int fl_axpy(int64_t n, double alpha, const double* x, double* y, fl_stream_t stream) {
  if (!x || !y) return fail(FL_E_VALUE, "null argument");
  k_axpy<<<grid_for(n, T), T, 0, (cudaStream_t)stream>>>(n, alpha, x, y);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fl_xpby(int64_t n, const double* x, double beta, double* y, fl_stream_t stream) {
  if (!x || !y) return fail(FL_E_VALUE, "null argument");
  k_xpby<<<grid_for(n, T), T, 0, (cudaStream_t)stream>>>(n, x, beta, y);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fl_pcg_step_init(int64_t n, const double* sigma1, const double* sigma2, const double* rhs, double* x,
                     double* r, double* p, double* out, fl_stream_t stream) {
  if (!sigma1 || !sigma2 || !rhs || !x || !r || !p || !out) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  int grid = 0;
  FL_TRY(pcg2_init(n, sigma1, sigma2, rhs, x, r, p, sc->partials, &grid, s));
  const int kinds[2] = {RED_SUM, RED_SUM};
  return reduce_fetch(sc, grid, 2, kinds, out, s);
}

int fl_pcg_step_update(int64_t n, const double* sigma1, const double* sigma2, double alpha, double* x, double* r,
                       const double* p, const double* g, double* out, fl_stream_t stream) {
  if (!sigma1 || !sigma2 || !x || !r || !p || !g || !out) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_pcg2_update_a<<<grid, T, 0, s>>>(n, sigma1, sigma2, alpha, nullptr, x, r, p, g, sc->partials);
  FL_LAUNCH_CHECK();
  const int kind = RED_SUM;
  return reduce_fetch(sc, grid, 1, &kind, out, s);
}

int fl_pcg_step_pupdate(int64_t n, const double* sigma1, const double* sigma2, const double* r, double beta,
                        double* p, double* out, fl_stream_t stream) {
  if (!sigma1 || !sigma2 || !r || !p || !out) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  int grid = 0;
  FL_TRY(pcg2_pupdate(n, sigma1, sigma2, r, beta, p, sc->partials, &grid, s));
  const int kind = RED_SUM;
  return reduce_fetch(sc, grid, 1, &kind, out, s);
}

int fl_pcg_step_alpha(const double* red2, const double* rho_dev, double* out_dev, fl_stream_t stream) {
  if (!red2 || !rho_dev || !out_dev) return fail(FL_E_VALUE, "null argument");
  k_step_alpha_dev<<<1, 32, 0, (cudaStream_t)stream>>>(red2, rho_dev, out_dev);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

// Device-scalar forms of the step-wise PCG (no host sync): the local partial
// goes to ``out_dev`` (device), alpha comes from device memory.
int fl_pcg_step_update_dev(int64_t n, const double* sigma1, const double* sigma2, const double* alpha_dev,
                           double* x, double* r, const double* p, const double* g, double* out_dev,
                           fl_stream_t stream) {
  if (!sigma1 || !sigma2 || !alpha_dev || !x || !r || !p || !g || !out_dev) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(n, T);
  k_pcg2_update_a<<<grid, T, 0, s>>>(n, sigma1, sigma2, 0.0, alpha_dev, x, r, p, g, sc->partials);
  FL_LAUNCH_CHECK();
  const int kind = RED_SUM;
  return finish_reduce(sc->partials, grid, 1, &kind, out_dev, s);
}

int fl_pcg_step_pupdate_dev(int64_t n, const double* sigma1, const double* sigma2, const double* r, double beta,
                            double* p, double* out_dev, fl_stream_t stream) {
  if (!sigma1 || !sigma2 || !r || !p || !out_dev) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  int grid = 0;
  FL_TRY(pcg2_pupdate(n, sigma1, sigma2, r, beta, p, sc->partials, &grid, s));
  const int kind = RED_SUM;
  return finish_reduce(sc->partials, grid, 1, &kind, out_dev, s);
}

int fl_objective_terms(int64_t n, const uint32_t* bits, const double* bhat, const double* x, int64_t n_beta,
                       const double* beta, double* out, fl_stream_t stream) {
  if (!bits || !bhat || !x || !out) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int grid = grid_for(std::max(n, n_beta), T);
  k_objective_terms<<<grid, T, 0, s>>>(n, bits, bhat, x, n_beta, beta, sc->partials);
  FL_LAUNCH_CHECK();
  const int kinds[2] = {RED_SUM, RED_SUM};
  return reduce_fetch(sc, grid, 2, kinds, out, s);
}

}  // extern "C"
