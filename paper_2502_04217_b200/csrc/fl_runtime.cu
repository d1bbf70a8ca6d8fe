// Runtime of libfftlasso_b200: error state, per-thread reduction scratch,
// deterministic reduction finish, plans (radix factorisation + twiddle
// tables), and the C-ABI entry points of the transform / observation / KKT
// operators.
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "fl_common.cuh"
#include "fl_internal.h"

namespace fl {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

// ---- reduction scratch, one per (host thread, device) ----
struct ScratchSet {
  Scratch s[kMaxDevices];
  ~ScratchSet() {
    // process teardown: the CUDA context may already be gone, ignore errors
    for (auto& x : s) {
      if (x.partials) cudaFree(x.partials);
      if (x.result) cudaFree(x.result);
      if (x.host) cudaFreeHost(x.host);
    }
  }
};
static thread_local ScratchSet g_scratch;

int scratch(Scratch** out) {
  int dev = 0;
  FL_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(FL_E_VALUE, "device index out of range");
  Scratch& s = g_scratch.s[dev];
  if (!s.partials) {
    if (cudaMalloc(&s.partials, sizeof(double) * kPartialSlots) != cudaSuccess ||
        cudaMalloc(&s.result, sizeof(double) * kResultSlots) != cudaSuccess ||
        cudaMallocHost(&s.host, sizeof(double) * kResultSlots) != cudaSuccess) {
      cudaGetLastError();
      return fail(FL_E_NOMEM, "cannot allocate reduction scratch");
    }
  }
  *out = &s;
  return FL_OK;
}

// One block per reduced row; fixed combine order -> deterministic.
__global__ void finish_kernel_kinds(const double* __restrict__ partials, int nblocks,
                                    unsigned long long kindbits, double* __restrict__ result) {
  __shared__ double red[32];
  const int row = blockIdx.x;
  const int kind = (int)((kindbits >> (2 * row)) & 3ull);
  const double* p = partials + (size_t)row * nblocks;
  double v = kind == RED_SUM ? 0.0 : (kind == RED_MAX ? -INFINITY : INFINITY);
  for (int i = threadIdx.x; i < nblocks; i += blockDim.x) {
    const double x = p[i];
    v = kind == RED_SUM ? v + x : (kind == RED_MAX ? PropMaxOp()(v, x) : PropMinOp()(v, x));
  }
  if (kind == RED_SUM) v = block_reduce(v, SumOp(), red);
  else if (kind == RED_MAX) v = block_reduce(v, PropMaxOp(), red);
  else v = block_reduce(v, PropMinOp(), red);
  if (threadIdx.x == 0) result[row] = v;
}

int finish_reduce(const double* partials, int nblocks, int nk, const int* kinds, double* result,
                  cudaStream_t stream) {
  if (nk > 32) return fail(FL_E_VALUE, "too many reduction rows");
  unsigned long long bits = 0;
  for (int k = 0; k < nk; ++k) bits |= (unsigned long long)(kinds[k] & 3) << (2 * k);
  finish_kernel_kinds<<<nk, 512, 0, stream>>>(partials, nblocks, bits, result);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int fetch_results(Scratch* s, int count, cudaStream_t stream) {
  FL_CUDA(cudaMemcpyAsync(s->host, s->result, sizeof(double) * count, cudaMemcpyDeviceToHost, stream));
  FL_CUDA(cudaStreamSynchronize(stream));
  return FL_OK;
}

// ---- plans ----
static std::vector<int> factor_radices(int m) {
  std::vector<int> r;
  while (m % 8 == 0) { r.push_back(8); m /= 8; }
  while (m % 4 == 0) { r.push_back(4); m /= 4; }
  while (m % 2 == 0) { r.push_back(2); m /= 2; }
  for (int p = 3; m > 1; p += 2) {
    while (m % p == 0) { r.push_back(p); m /= p; }
    if ((int64_t)p * p > m && m > 1) { r.push_back(m); m = 1; }
  }
  return r;
}

static int make_axis_plan(fl_plan* p, int m, AxisPlan& ap) {
  ap.m = m;
  std::vector<int> r = factor_radices(m);
  if ((int)r.size() > kMaxStages) return fail(FL_E_SHAPE, "too many radix stages");
  ap.nst = (int)r.size();
  for (int i = 0; i < ap.nst; ++i) ap.radix[i] = r[i];
  // twiddles exp(-2 pi i k / m) in extended precision; exact at the quarter turns
  std::vector<double2> tw(m);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int k = 0; k < m; ++k) {
    const long double ang = two_pi * (long double)k / (long double)m;
    tw[k].x = (double)cosl(ang);
    tw[k].y = (double)(-sinl(ang));
    if ((int64_t)4 * k % m == 0) {
      const int q = (int)((int64_t)4 * k / m);
      const double c[4] = {1.0, 0.0, -1.0, 0.0}, s[4] = {0.0, -1.0, 0.0, 1.0};
      tw[k].x = c[q];
      tw[k].y = s[q];
    }
  }
  void* d = nullptr;
  FL_CUDA(cudaMalloc(&d, sizeof(double2) * m));
  p->owned.push_back(d);
  FL_CUDA(cudaMemcpy(d, tw.data(), sizeof(double2) * m, cudaMemcpyHostToDevice));
  ap.tw = static_cast<const double2*>(d);
  return FL_OK;
}

// Largest axis the single-CTA shared-memory engines handle: power-of-two
// lengths up to 8192 (register engine), others while two fibre buffers fit.
static bool fits_one_cta(int m) {
  if (m <= 8192 && (m & (m - 1)) == 0) return true;
  return 2 * (m + 1) * 16 <= 226 * 1024;
}

static int build_axis(fl_plan* p, int a) {
  const int m = (int)p->dims[a];
  FL_TRY(make_axis_plan(p, m, p->axis[a]));
  if (fits_one_cta(m)) return FL_OK;
  LongAxis& la = p->lng[a];
  FL_TRY(long_factor(m, &la.m1, &la.m2));
  FL_TRY(make_axis_plan(p, la.m1, la.p1));
  FL_TRY(make_axis_plan(p, la.m2, la.p2));
  // fibre pairs of this axis times m complex entries
  int64_t pairs = p->n / m / 2;
  if (pairs < 1) pairs = 1;
  void* d = nullptr;
  FL_CUDA(cudaMalloc(&d, sizeof(double2) * (size_t)pairs * m));
  p->owned.push_back(d);
  la.scratch = static_cast<double2*>(d);
  la.on = true;
  return FL_OK;
}

}  // namespace fl

using namespace fl;

extern "C" {

int fl_version(void) { return 1; }

const char* fl_last_error(void) { return g_err.c_str(); }

int fl_plan_create(int ndim, const int64_t* dims, int device, fl_plan_t* out) {
  return fl_plan_create_ex(ndim, dims, (1 << ndim) - 1, device, out);
}

int fl_plan_create_ex(int ndim, const int64_t* dims, int transform_axes, int device, fl_plan_t* out) {
  if (!out) return fail(FL_E_VALUE, "null output");
  *out = nullptr;
  if (ndim < 1 || ndim > 3) return fail(FL_E_SHAPE, "need 1 to 3 axes, got " + std::to_string(ndim));
  int64_t n = 1;
  for (int a = 0; a < ndim; ++a) {
    const bool tr = (transform_axes >> a) & 1;
    if (tr && (dims[a] < 2 || dims[a] % 2))
      return fail(FL_E_SHAPE, "every axis must be even and >= 2, got " + std::to_string(dims[a]));
    if (!tr && dims[a] < 1) return fail(FL_E_SHAPE, "batch extent must be >= 1");
    if (dims[a] > (1 << 30)) return fail(FL_E_SHAPE, "axis too long");
    n *= dims[a];
  }
  FL_CUDA(cudaSetDevice(device));
  fl_plan* p = new fl_plan();
  p->ndim = ndim;
  p->n = n;
  p->device = device;
  for (int a = 0; a < ndim; ++a) p->dims[a] = dims[a];
  for (int a = 0; a < ndim; ++a) {
    p->planned[a] = (transform_axes >> a) & 1;
    if (!p->planned[a]) continue;
    int st = build_axis(p, a);
    if (st != FL_OK) {
      fl_plan_destroy(p);
      return st;
    }
  }
  *out = p;
  return FL_OK;
}

int fl_plan_destroy(fl_plan_t p) {
  if (!p) return FL_OK;
  pcg_graphs_release(p);
  for (void* d : p->owned) cudaFree(d);
  delete p;
  return FL_OK;
}

int64_t fl_plan_n(fl_plan_t p) { return p ? p->n : -1; }

int fl_synthesize(fl_plan_t p, const double* beta, double* x, fl_stream_t stream) {
  if (!p || !beta || !x) return fail(FL_E_VALUE, "null argument");
  return op_synthesize(p, beta, x, (cudaStream_t)stream);
}

int fl_analyze(fl_plan_t p, const double* x, double* beta, fl_stream_t stream) {
  if (!p || !beta || !x) return fail(FL_E_VALUE, "null argument");
  return op_analyze(p, x, beta, (cudaStream_t)stream);
}

int fl_axis_pass(fl_plan_t p, int axis, int analysis, const double* in, double* out, fl_stream_t stream) {
  if (!p || !in || !out) return fail(FL_E_VALUE, "null argument");
  if (axis < 0 || axis >= p->ndim) return fail(FL_E_VALUE, "axis out of range");
  const int kind = analysis ? K_ANALYZE : K_SYNTH;
  return run_pass(p, axis, kind, in, out, nullptr, nullptr, nullptr, nullptr, (cudaStream_t)stream);
}

int fl_fused_mask_pass(fl_plan_t p, const uint32_t* bits, const double* bhat, const double* in, double* out,
                       double* nrm_host, fl_stream_t stream) {
  if (!p || !bits || !in || !out) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int last = p->ndim - 1;
  const bool want = nrm_host && !bhat;
  if (want && p->lng[last].on) return fail(FL_E_VALUE, "norm output not available on four-step axes");
  Scratch* sc = nullptr;
  FL_TRY(scratch(&sc));
  int nb = 0;
  FL_TRY(run_pass_n(p, last, bhat ? K_RESID : K_GRAM, in, out, bits, bhat, nullptr, &nb,
                    want ? sc->partials : nullptr, s));
  if (want) {
    const int kind = RED_SUM;
    FL_TRY(finish_reduce(sc->partials, nb, 1, &kind, sc->result, s));
    FL_TRY(fetch_results(sc, 1, s));
    *nrm_host = sc->host[0];
  }
  return FL_OK;
}

int fl_fused_mask_pass_dev(fl_plan_t p, const uint32_t* bits, const double* in, double* out, double* nrm_dev,
                           fl_stream_t stream) {
  if (!p || !bits || !in || !out || !nrm_dev) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int last = p->ndim - 1;
  if (p->lng[last].on) return fail(FL_E_VALUE, "norm output not available on four-step axes");
  Scratch* sc = nullptr;
  FL_TRY(scratch(&sc));
  int nb = 0;
  FL_TRY(run_pass_n(p, last, K_GRAM, in, out, bits, nullptr, nullptr, &nb, sc->partials, s));
  const int kind = RED_SUM;
  return finish_reduce(sc->partials, nb, 1, &kind, nrm_dev, s);
}

int fl_gram(fl_plan_t p, const uint32_t* bits, const double* beta, double* out, fl_stream_t stream) {
  if (!p || !bits || !beta || !out) return fail(FL_E_VALUE, "null argument");
  return op_gram(p, bits, nullptr, false, beta, out, nullptr, nullptr, (cudaStream_t)stream);
}

int fl_residual_adjoint(fl_plan_t p, const uint32_t* bits, const double* bhat, const double* beta,
                        double* out, fl_stream_t stream) {
  if (!p || !bits || !bhat || !out) return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (!beta) {
    FL_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * p->n, s));
    beta = out;
  }
  return op_gram(p, bits, bhat, true, beta, out, nullptr, nullptr, s);
}

int fl_kkt_apply(fl_plan_t p, const uint32_t* bits, const double* sigma1, const double* sigma2,
                 const double* d_beta, const double* d_z, double* top, double* bottom,
                 double* pkp_host, fl_stream_t stream) {
  if (!p || !bits || !sigma1 || !sigma2 || !d_beta || !d_z || !top)
    return fail(FL_E_VALUE, "null argument");
  if (top == d_beta || top == d_z) return fail(FL_E_VALUE, "top must not alias the direction");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc = nullptr;
  FL_TRY(scratch(&sc));
  KktEpi e;
  e.pb = d_beta;
  e.pz = d_z;
  e.sig1 = sigma1;
  e.sig2 = sigma2;
  e.bottom = bottom;
  e.partials = pkp_host ? sc->partials : nullptr;
  int nb = 0;
  FL_TRY(op_gram(p, bits, nullptr, false, d_beta, top, &e, &nb, s));
  if (pkp_host) {
    const int kind = RED_SUM;
    FL_TRY(finish_reduce(sc->partials, nb, 1, &kind, sc->result, s));
    FL_TRY(fetch_results(sc, 1, s));
    *pkp_host = sc->host[0];
  }
  return FL_OK;
}

int fl_kkt_epilogue(int64_t n, double* g, const double* d_beta, const double* d_z, const double* sigma1,
                    const double* sigma2, double* bottom, double* pkp_host, fl_stream_t stream) {
  if (!g || !d_beta || !d_z || !sigma1 || !sigma2) return fail(FL_E_VALUE, "null argument");
  if (n % 2) return fail(FL_E_SHAPE, "epilogue needs an even length");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  int nb = 0;
  FL_TRY(kkt_epilogue(n, g, d_beta, d_z, sigma1, sigma2, bottom, pkp_host ? sc->partials : nullptr, &nb, s));
  if (pkp_host) {
    const int kind = RED_SUM;
    FL_TRY(finish_reduce(sc->partials, nb, 1, &kind, sc->result, s));
    FL_TRY(fetch_results(sc, 1, s));
    *pkp_host = sc->host[0];
  }
  return FL_OK;
}

int fl_kkt_order(fl_plan_t p) { return p && kkt_order_b(p) ? 1 : 0; }

int fl_kkt_apply_profiled(fl_plan_t p, const uint32_t* bits, const double* sigma1,
                          const double* sigma2, const double* d_beta, const double* d_z, double* top,
                          double* bottom, double* pass_ms, int* npasses, fl_stream_t stream) {
  if (!p || !bits || !sigma1 || !sigma2 || !d_beta || !d_z || !top || !pass_ms || !npasses)
    return fail(FL_E_VALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int d = p->ndim;
  const int np = 2 * d;  // at most 2d-1 transform passes + the elementwise epilogue
  cudaEvent_t ev[8];
  for (int i = 0; i <= np; ++i) FL_CUDA(cudaEventCreate(&ev[i]));
  int st = FL_OK;
  FL_CUDA(cudaEventRecord(ev[0], s));
  int k = 0;
  if (kkt_order_b(p)) {  // same order as fl_kkt_apply (op_gram)
    const double* src = d_beta;
    for (int a = d - 1; a >= 1 && st == FL_OK; --a) {
      st = run_pass(p, a, K_SYNTH, src, top, nullptr, nullptr, nullptr, nullptr, s);
      cudaEventRecord(ev[++k], s);
      src = top;
    }
    if (st == FL_OK) st = run_pass(p, 0, K_GRAM, top, top, bits, nullptr, nullptr, nullptr, s);
    cudaEventRecord(ev[++k], s);
    KktEpi e;
    e.pb = d_beta;
    e.pz = d_z;
    e.sig1 = sigma1;
    e.sig2 = sigma2;
    e.bottom = bottom;
    for (int a = 1; a < d && st == FL_OK; ++a) {
      st = run_pass(p, a, K_ANALYZE, top, top, nullptr, nullptr, a == d - 1 ? &e : nullptr, nullptr, s);
      cudaEventRecord(ev[++k], s);
    }
  } else if (d == 1) {
    st = run_pass(p, 0, K_GRAM, d_beta, top, bits, nullptr, nullptr, nullptr, s);
    cudaEventRecord(ev[++k], s);
  } else {
    const double* src = d_beta;
    for (int a = 0; a < d - 1 && st == FL_OK; ++a) {
      st = run_pass(p, a, K_SYNTH, src, top, nullptr, nullptr, nullptr, nullptr, s);
      cudaEventRecord(ev[++k], s);
      src = top;
    }
    if (st == FL_OK) st = run_pass(p, d - 1, K_GRAM, top, top, bits, nullptr, nullptr, nullptr, s);
    cudaEventRecord(ev[++k], s);
    for (int a = d - 2; a >= 0 && st == FL_OK; --a) {
      st = run_pass(p, a, K_ANALYZE, top, top, nullptr, nullptr, nullptr, nullptr, s);
      cudaEventRecord(ev[++k], s);
    }
  }
  if (!kkt_order_b(p)) {
    if (st == FL_OK) st = kkt_epilogue(p->n, top, d_beta, d_z, sigma1, sigma2, bottom, nullptr, nullptr, s);
    cudaEventRecord(ev[++k], s);
  }
  if (st == FL_OK) {
    FL_CUDA(cudaEventSynchronize(ev[k]));
    for (int i = 0; i < k; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      pass_ms[i] = ms;
    }
    *npasses = k;
  }
  for (int i = 0; i <= np; ++i) cudaEventDestroy(ev[i]);
  return st;
}

}  // extern "C"
