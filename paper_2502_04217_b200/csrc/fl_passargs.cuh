// Pass arguments and fibre-pair geometry shared by the generic
// (fl_pass.cu) and register-resident (fl_fastpass.cu) axis-pass kernels.
#pragma once

#include "fl_common.cuh"
#include "fl_internal.h"

namespace fl {

struct PassArgs {
  const double* in;
  double* out;
  int64_t G;      // fibre pairs
  int64_t inner;  // strided: element stride (doubles); also pairs-per-outer * 2
  int m, h;
  int has_y;
  int F, fs;
  double c0, c1;  // 1/sqrt(m), 1/sqrt(2m)
  AxisPlan plan;
  const uint32_t* bits;
  const double* bhat;
  KktEpi epi;
  double* nrm_partials;  // K_GRAM: per-block ||Z A beta||^2 partials (nullable)
};

// Geometry of fibre pair g: element k of fibre x at bx + k*st, of y at by + k*st.
struct Geo {
  int64_t bx, by, st;
};

template <bool STRIDED>
__device__ __forceinline__ Geo geo(const PassArgs& A, int64_t g) {
  Geo r;
  if (STRIDED) {
    const int64_t ppo = A.inner >> 1;
    int64_t o, q;
    if (A.G <= 0xffffffffLL) {  // 32-bit division (all single-GPU grid sizes)
      const unsigned o32 = (unsigned)g / (unsigned)ppo;
      o = o32;
      q = g - (int64_t)o32 * ppo;
    } else {
      o = g / ppo;
      q = g - o * ppo;
    }
    r.bx = o * (int64_t)A.m * A.inner + 2 * q;
    r.by = r.bx + 1;
    r.st = A.inner;
  } else {
    r.bx = A.has_y ? 2 * g * (int64_t)A.m : g * (int64_t)A.m;
    r.by = A.has_y ? r.bx + A.m : -1;
    r.st = 1;
  }
  return r;
}

__device__ __forceinline__ bool missing(const uint32_t* bits, int64_t v) {
  return (__ldg(bits + (v >> 5)) >> (v & 31)) & 1u;
}

// KKT epilogue at voxel v with gram value gv (NumPy order, no FMA).
__device__ __forceinline__ void kkt_store(const PassArgs& A, int64_t v, double gv, double& acc) {
  const double pb = A.epi.pb[v], pz = A.epi.pz[v];
  const double s1 = A.epi.sig1[v], s2 = A.epi.sig2[v];
  const double l1 = add(s1, s2), l2 = sub(s1, s2);
  const double top = add(add(gv, mul(l1, pb)), mul(l2, pz));
  const double bot = add(mul(l2, pb), mul(l1, pz));
  A.out[v] = top;
  if (A.epi.bottom) A.epi.bottom[v] = bot;
  acc += pb * top + pz * bot;
}

template <bool STRIDED, bool EPI>
__device__ __forceinline__ void put(const PassArgs& A, int64_t v, double val, double& acc) {
  if (EPI) kkt_store(A, v, val, acc);
  else A.out[v] = val;
}


using KernelFn = void (*)(const PassArgs);

int launch_fast(int m, bool strided, int kind, bool epi, const PassArgs& A, int* nblocks,
                cudaStream_t s);
bool fast_supported(int m);

}  // namespace fl
