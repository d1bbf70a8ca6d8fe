// Device-resident PCG on the condensed KKT system (pcg.py:57-127 applied as
// in ipm.py:318-327).  Per iteration (v2, default): the gram g = G p_beta
// (2d-1 HBM passes; the fused mask pass also reduces ||Z A p_beta||^2, the
// matrix part of p.Kp), one fused x/r/P^{-1}/rho pass that forms K p in
// registers from g, and one p-update pass that also reduces the diagonal
// part of the next p.Kp.  The dot products finish on device and are read back
// with a single stream sync per iteration -- the only host round trip.
// Scalar recurrences (alpha, beta, the stopping test, breakdown checks)
// follow pcg.py exactly, in IEEE double.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "fl_common.cuh"
#include "fl_internal.h"

using namespace fl;

namespace {

constexpr int64_t kPcgIterCap = 5000;  // pcg.py:19

struct History {
  double* buf;
  int64_t cap, n = 0;
  void operator()(double v) {
    if (buf && n < cap) buf[n] = v;
    ++n;
  }
};

int check_rho(double rho, int64_t k) {
  if (!std::isfinite(rho) || rho < 0)
    return fail(FL_E_BREAKDOWN, k == 0 ? "preconditioner produced r'P^{-1}r = " + std::to_string(rho)
                                       : "r'P^{-1}r = " + std::to_string(rho) + " at iteration " +
                                             std::to_string(k));
  return FL_OK;
}

int check_curv(double curv, int64_t k) {
  if (!std::isfinite(curv) || curv <= 0)
    return fail(FL_E_BREAKDOWN, "nonpositive curvature p'Kp = " + std::to_string(curv) + " at iteration " +
                                    std::to_string(k));
  return FL_OK;
}

// v2 (default): curvature p.Kp = ||Z A p_beta||^2 (reduced inside the fused gram
// pass) + the diagonal form accumulated where p is written; the update pass
// reads g = G p_beta and forms K p in registers, so K p never touches HBM.
// Per iteration: 2d-1 transform passes + update (104 B/voxel) + p-update
// (64 B/voxel) = 248 B/voxel in 3D, vs 280 for v1.
int pcg_v2(fl_plan_t p, const uint32_t* bits, const double* sigma1, const double* sigma2, const double* rhs,
           double* x, double* work, double abs_tol, double rel_tol, int64_t max_iters, fl_pcg_result* res,
           double* history, int64_t max_history, cudaStream_t s) {
  const int64_t n = p->n;
  double* r = work;
  double* pv = work + 2 * n;
  double* gp = work + 4 * n;
  double* slots = work + 6 * n;  // [rho_a, rho_b, curv_G, curv_diag]
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int64_t limit = max_iters >= 0 ? max_iters : std::min<int64_t>(10 * 2 * n, kPcgIterCap);
  const int sum2[2] = {RED_SUM, RED_SUM};
  History record{history, max_history};
  int nb = 0;
  FL_TRY(pcg2_init(n, sigma1, sigma2, rhs, x, r, pv, sc->partials, &nb, s));
  // rows: rho -> slot 0, diag form -> slot 3 (finish writes rows contiguously)
  FL_TRY(finish_reduce(sc->partials, nb, 2, sum2, sc->result, s));
  FL_CUDA(cudaMemcpyAsync(slots, sc->result, sizeof(double), cudaMemcpyDeviceToDevice, s));
  FL_CUDA(cudaMemcpyAsync(slots + 3, sc->result + 1, sizeof(double), cudaMemcpyDeviceToDevice, s));
  FL_CUDA(cudaMemcpyAsync(sc->host, slots, sizeof(double), cudaMemcpyDeviceToHost, s));
  FL_CUDA(cudaStreamSynchronize(s));
  double rho = sc->host[0];
  FL_TRY(check_rho(rho, 0));
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
  const int ksum = RED_SUM;
  for (int64_t k = 1; k <= limit; ++k) {
    int nbg = 0, nbu = 0, nbp = 0;
    bool have_norm = false;
    FL_TRY(op_gram_norm(p, bits, pv, gp, sc->partials, &nbg, &have_norm, s));
    if (!have_norm) FL_TRY(dot_partials(n, pv, gp, sc->partials, &nbg, s));
    FL_TRY(finish_reduce(sc->partials, nbg, 1, &ksum, slots + 2, s));
    FL_TRY(pcg2_update(n, sigma1, sigma2, slots + cur, slots + 2, slots + 3, x, r, pv, gp, sc->partials, &nbu, s));
    FL_TRY(finish_reduce(sc->partials, nbu, 1, &ksum, slots + (1 - cur), s));
    FL_CUDA(cudaMemcpyAsync(sc->host, slots, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    const double curv = sc->host[2] + sc->host[3];
    FL_TRY(check_curv(curv, k));
    const double rho_next = sc->host[1 - cur];
    FL_TRY(check_rho(rho_next, k));
    norm = std::sqrt(rho_next);
    record(norm);
    if (norm <= thr) {
      res->iterations = k;
      res->converged = 1;
      res->residual_norm = norm;
      return FL_OK;
    }
    const double beta = rho_next / rho;
    FL_TRY(pcg2_pupdate(n, sigma1, sigma2, r, beta, pv, sc->partials, &nbp, s));
    FL_TRY(finish_reduce(sc->partials, nbp, 1, &ksum, slots + 3, s));
    rho = rho_next;
    cur = 1 - cur;
  }
  res->iterations = limit;
  res->converged = 0;
  res->residual_norm = norm;
  return FL_OK;
}


// v1: materialised K p (gram + elementwise epilogue with d.Kd partials), then
// a fused update pass reading K p; kept behind FL_PCG_V1=1 for comparison.
int pcg_v1(fl_plan_t p, const uint32_t* bits, const double* sigma1, const double* sigma2, const double* rhs,
           double* x, double* work, double abs_tol, double rel_tol, int64_t max_iters, fl_pcg_result* res,
           double* history, int64_t max_history, cudaStream_t s) {
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
  History record{history, max_history};
  int nb = 0;
  FL_TRY(pcg_init(n, sigma1, sigma2, rhs, x, r, pv, sc->partials, &nb, s));
  FL_TRY(finish_reduce(sc->partials, nb, 1, &ksum, slots, s));
  FL_CUDA(cudaMemcpyAsync(sc->host, slots, sizeof(double), cudaMemcpyDeviceToHost, s));
  FL_CUDA(cudaStreamSynchronize(s));
  double rho = sc->host[0];
  FL_TRY(check_rho(rho, 0));
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
    FL_TRY(pcg_update(n, sigma1, sigma2, slots + cur, slots + 2, x, r, pv, kt, kb, sc->partials, &nbu, s));
    FL_TRY(finish_reduce(sc->partials, nbu, 1, &ksum, slots + (1 - cur), s));
    FL_CUDA(cudaMemcpyAsync(sc->host, slots, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    FL_TRY(check_curv(sc->host[2], k));
    const double rho_next = sc->host[1 - cur];
    FL_TRY(check_rho(rho_next, k));
    norm = std::sqrt(rho_next);
    record(norm);
    if (norm <= thr) {
      res->iterations = k;
      res->converged = 1;
      res->residual_norm = norm;
      return FL_OK;
    }
    FL_TRY(pcg_pupdate(n, sigma1, sigma2, r, rho_next / rho, pv, s));
    rho = rho_next;
    cur = 1 - cur;
  }
  res->iterations = limit;
  res->converged = 0;
  res->residual_norm = norm;
  return FL_OK;
}

}  // namespace

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
  static const bool v1 = [] {
    const char* e = std::getenv("FL_PCG_V1");
    return e && e[0] == '1';
  }();
  auto* run = v1 ? pcg_v1 : pcg_v2;
  return run(p, bits, sigma1, sigma2, rhs, x, work, abs_tol, rel_tol, max_iters, res, history, max_history,
             (cudaStream_t)stream);
}

}  // extern "C"
