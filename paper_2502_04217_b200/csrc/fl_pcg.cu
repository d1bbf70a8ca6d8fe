// Device-resident PCG on the condensed KKT system (pcg.py:57-127 applied as
// in ipm.py:318-327).  Per iteration: one fused gram + KKT-epilogue matvec
// (2d-1 HBM passes, d.Kd partials in the last pass), one fused
// x/r/preconditioner/rho pass, and one p-update pass; the two dot products
// finish on device and are read back with a single stream sync, which is
// the only host round trip.  Scalar recurrences (alpha, beta, the stopping
// test, breakdown checks) follow pcg.py exactly, in IEEE double.
#include <cmath>
#include <string>

#include "fl_common.cuh"
#include "fl_internal.h"

using namespace fl;

namespace {
constexpr int64_t kPcgIterCap = 5000;  // pcg.py:19
}

extern "C" {

int64_t fl_pcg_work_doubles(int64_t n) { return 6 * n + 16; }

int fl_pcg_kkt(fl_plan_t p, const uint32_t* bits, const double* sigma1, const double* sigma2,
               const double* rhs, double* x, double* work, double abs_tol, double rel_tol,
               int64_t max_iters, fl_pcg_result* res, double* history, int64_t max_history,
               fl_stream_t stream) {
  if (!p || !bits || !sigma1 || !sigma2 || !rhs || !x || !work || !res)
    return fail(FL_E_VALUE, "null argument");
  if (abs_tol < 0 || rel_tol < 0) return fail(FL_E_VALUE, "tolerances must be nonnegative");
  if (abs_tol == 0 && rel_tol == 0) return fail(FL_E_VALUE, "abs_tol and rel_tol cannot both be zero");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = p->n;
  double* r = work;
  double* pv = work + 2 * n;
  double* kt = work + 4 * n;
  double* kb = work + 5 * n;
  double* slots = work + 6 * n;  // [rho_a, rho_b, curv]
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int64_t limit = max_iters >= 0 ? max_iters : std::min<int64_t>(10 * 2 * n, kPcgIterCap);
  const int ksum = RED_SUM;
  int64_t nh = 0;
  auto record = [&](double v) {
    if (history && nh < max_history) history[nh] = v;
    ++nh;
  };

  int nb = 0;
  FL_TRY(pcg_init(n, sigma1, sigma2, rhs, x, r, pv, sc->partials, &nb, s));
  FL_TRY(finish_reduce(sc->partials, nb, 1, &ksum, slots, s));
  FL_CUDA(cudaMemcpyAsync(sc->host, slots, sizeof(double), cudaMemcpyDeviceToHost, s));
  FL_CUDA(cudaStreamSynchronize(s));
  double rho = sc->host[0];
  if (!std::isfinite(rho) || rho < 0)
    return fail(FL_E_BREAKDOWN, "preconditioner produced r'P^{-1}r = " + std::to_string(rho));
  const double norm0 = std::sqrt(rho);
  const double thr = abs_tol + rel_tol * norm0;
  record(norm0);
  res->norm0 = norm0;
  if (norm0 <= thr) {
    res->iterations = 0;
    res->converged = 1;
    res->residual_norm = norm0;
    return FL_OK;
  }
  double norm = norm0;
  int cur = 0;
  KktEpi e;
  e.pb = pv;
  e.pz = pv + n;
  e.sig1 = sigma1;
  e.sig2 = sigma2;
  e.bottom = kb;
  e.partials = sc->partials;
  for (int64_t k = 1; k <= limit; ++k) {
    int nbk = 0, nbu = 0;
    FL_TRY(op_gram(p, bits, nullptr, false, pv, kt, &e, &nbk, s));
    FL_TRY(finish_reduce(sc->partials, nbk, 1, &ksum, slots + 2, s));
    // partials are reused by the update pass only after finish has consumed them (stream order)
    FL_TRY(pcg_update(n, sigma1, sigma2, slots + cur, slots + 2, x, r, pv, kt, kb, sc->partials, &nbu, s));
    FL_TRY(finish_reduce(sc->partials, nbu, 1, &ksum, slots + (1 - cur), s));
    FL_CUDA(cudaMemcpyAsync(sc->host, slots, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    const double curv = sc->host[2];
    if (!std::isfinite(curv) || curv <= 0)
      return fail(FL_E_BREAKDOWN, "nonpositive curvature p'Kp = " + std::to_string(curv) +
                                      " at iteration " + std::to_string(k));
    const double rho_next = sc->host[1 - cur];
    if (!std::isfinite(rho_next) || rho_next < 0)
      return fail(FL_E_BREAKDOWN, "r'P^{-1}r = " + std::to_string(rho_next) + " at iteration " +
                                      std::to_string(k));
    norm = std::sqrt(rho_next);
    record(norm);
    if (norm <= thr) {
      res->iterations = k;
      res->converged = 1;
      res->residual_norm = norm;
      return FL_OK;
    }
    const double beta = rho_next / rho;
    FL_TRY(pcg_pupdate(n, sigma1, sigma2, r, beta, pv, s));
    rho = rho_next;
    cur = 1 - cur;
  }
  res->iterations = limit;
  res->converged = 0;
  res->residual_norm = norm;
  return FL_OK;
}

}  // extern "C"
