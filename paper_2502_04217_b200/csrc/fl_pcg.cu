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
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <string>
#include <mutex>
#include <vector>

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
// Reduce the start partials (rows: rho, diagonal curvature[, interior flag])
// into slots[0] / slots[3] and read rho (and the flag) back: the one host sync
// before the loop.
int pcg_start_fetch(Scratch* sc, int nb, bool with_flag, double* slots, double* rho, double* flag,
                    cudaStream_t s) {
  const int kinds[3] = {RED_SUM, RED_SUM, RED_MAX};
  FL_TRY(finish_reduce(sc->partials, nb, with_flag ? 3 : 2, kinds, sc->result, s));
  FL_CUDA(cudaMemcpyAsync(slots, sc->result, sizeof(double), cudaMemcpyDeviceToDevice, s));
  FL_CUDA(cudaMemcpyAsync(slots + 3, sc->result + 1, sizeof(double), cudaMemcpyDeviceToDevice, s));
  FL_CUDA(cudaMemcpyAsync(sc->host, sc->result, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  FL_CUDA(cudaStreamSynchronize(s));
  *rho = sc->host[0];
  if (flag) *flag = with_flag ? sc->host[2] : 0.0;
  return FL_OK;
}

// v2 loop from a started state (x = 0, r = rhs, p = P^{-1} r; slots[0] = rho,
// slots[3] = diagonal curvature).
int pcg_v2_loop(fl_plan_t p, const uint32_t* bits, const double* sigma1, const double* sigma2, double* x,
                double* work, double rho, double abs_tol, double rel_tol, int64_t limit, fl_pcg_result* res,
                double* history, int64_t max_history, cudaStream_t s) {
  const int64_t n = p->n;
  double* r = work;
  double* pv = work + 2 * n;
  double* gp = work + 4 * n;
  double* slots = work + 6 * n;  // [rho_a, rho_b, curv_G, curv_diag]
  Scratch* sc;
  FL_TRY(scratch(&sc));
  History record{history, max_history};
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

// v2 (host loop): curvature p.Kp = ||Z A p_beta||^2 (reduced inside the fused
// gram pass) + the diagonal form accumulated where p is written; the update
// pass reads g = G p_beta and forms K p in registers, so K p never touches
// HBM.  Per iteration: 2d-1 transform passes + update (104 B/voxel) +
// p-update (64 B/voxel) = 248 B/voxel in 3D, vs 280 for v1.
int pcg_v2(fl_plan_t p, const uint32_t* bits, const double* sigma1, const double* sigma2, const double* rhs,
           double* x, double* work, double abs_tol, double rel_tol, int64_t limit, fl_pcg_result* res,
           double* history, int64_t max_history, cudaStream_t s) {
  const int64_t n = p->n;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  int nb = 0;
  double rho = 0.0;
  FL_TRY(pcg2_init(n, sigma1, sigma2, rhs, x, work, work + 2 * n, sc->partials, &nb, s));
  FL_TRY(pcg_start_fetch(sc, nb, false, work + 6 * n, &rho, nullptr, s));
  return pcg_v2_loop(p, bits, sigma1, sigma2, x, work, rho, abs_tol, rel_tol, limit, res, history, max_history, s);
}

// ---------------------------------------------------------------------------
// v3 (default when no host history is requested): the v2 iteration captured
// once per (plan, operands) into a CUDA graph whose WHILE conditional node
// loops on the device.  A one-thread control kernel after the update pass
// performs pcg.py's scalar step (breakdown checks, the stopping test, beta)
// and clears the loop condition, so a whole PCG solve is ONE graph launch and
// ONE host sync instead of one sync per iteration.  Same kernels, same
// operands, same scalar arithmetic (IEEE sqrt / divide) as v2.
// ---------------------------------------------------------------------------

struct PcgCtl {      // at work + 6n + 8 (8 doubles)
  double thr;        // stopping threshold abs_tol + rel_tol * ||r0||_P
  double norm;       // last preconditioned residual norm
  double bad;        // offending value of a breakdown
  long long limit;   // iteration cap
  long long k;       // iterations done
  int status;        // 0 running, 1 converged, 2 cap reached, 3 curvature, 4 r'P^{-1}r breakdown,
                     // 5 non-interior state (gated graph only)
  int done;
  double abs_tol;    // gated graph: thr is formed on the device from these
  double rel_tol;
};
static_assert(sizeof(PcgCtl) <= 8 * sizeof(double), "PcgCtl must fit its work slots");

// slots: [rho, rho_next, curv_G, curv_diag, beta]
__global__ void k_pcg_control(PcgCtl* __restrict__ c, double* __restrict__ slots,
                              cudaGraphConditionalHandle h) {
  if (threadIdx.x != 0) return;
  if (c->done) {
    cudaGraphSetConditional(h, 0);
    return;
  }
  const long long k = ++c->k;
  const double curv = slots[2] + slots[3];
  const double rn = slots[1];
  int st = 0;
  double bad = 0.0;
  if (!isfinite(curv) || curv <= 0) {
    st = 3;
    bad = curv;
  } else if (!isfinite(rn) || rn < 0) {
    st = 4;
    bad = rn;
  } else {
    const double norm = sqrt(rn);
    c->norm = norm;
    if (norm <= c->thr) {
      st = 1;
    } else if (k >= c->limit) {
      st = 2;
    } else {
      slots[4] = rn / slots[0];  // beta = rz_new / rz (pcg.py)
      slots[0] = rn;
    }
  }
  if (st) {
    c->status = st;
    c->bad = bad;
    c->done = 1;
    cudaGraphSetConditional(h, 0);
  }
}

// Gate ahead of the WHILE node (gated graph of fl_ipm_newton_step): the PCG
// start check done on the device instead of pcg_start_fetch's host sync --
// res = reduced start partials [rho, diagonal curvature, interior flag].
// Same tests in the same order as the host (interior flag, r'P^{-1}r, then
// ||r0|| <= thr), thr = abs_tol + rel_tol * sqrt(rho) rounded as on the host
// (no contraction).  Opens the loop only when there is work to do.
__global__ void k_pcg_gate(PcgCtl* __restrict__ c, const double* __restrict__ res, double* __restrict__ slots,
                           double* __restrict__ dev, cudaGraphConditionalHandle h) {
  if (threadIdx.x != 0) return;
  const double rho = res[0];
  slots[0] = rho;
  slots[3] = res[1];
  int st = 0;
  double bad = 0.0;
  dev[12] = NAN;
  if (res[2] != 0.0) {
    st = 5;
  } else if (!isfinite(rho) || rho < 0) {
    st = 4;
    bad = rho;
  } else {
    const double norm0 = sqrt(rho);
    dev[12] = norm0;
    c->norm = norm0;
    c->thr = __dadd_rn(c->abs_tol, __dmul_rn(c->rel_tol, norm0));
    if (norm0 <= c->thr) st = 1;
    else if (c->limit <= 0) st = 2;
  }
  c->k = 0;
  c->bad = bad;
  c->status = st;
  c->done = st != 0;
  cudaGraphSetConditional(h, st == 0 ? 1 : 0);
}

// PCG verdict into the step record (fl_ipm_newton_step): dev[8..12].
__global__ void k_step_pack(const PcgCtl* __restrict__ c, double norm0, double* __restrict__ dev) {
  if (threadIdx.x != 0) return;
  dev[8] = (double)c->status;
  dev[9] = (double)c->k;
  dev[10] = c->norm;
  dev[11] = c->bad;
  if (norm0 >= 0.0) dev[12] = norm0;  // < 0: written by the gate
}

// A captured graph bakes in every pointer it touches: the operands AND the
// calling thread's reduction scratch (partials, result), so all of them are
// the key.  Bounded LRU per plan (kPcgGraphCap entries); an evicted exec that
// is still in flight is freed by the driver when it completes.
struct PcgGraph {
  const uint32_t* bits;
  const double *sig1, *sig2;
  double *x, *work;
  const double *partials, *result;
  bool gated;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

constexpr size_t kPcgGraphCap = 4;

struct PcgGraphs {
  std::vector<PcgGraph> v;  // least recently used first
  cudaStream_t capture = nullptr;
  std::mutex mu;
};

void destroy_graph(PcgGraph& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  if (g.graph) cudaGraphDestroy(g.graph);
  g.exec = nullptr;
  g.graph = nullptr;
}

// Enqueue one v2 iteration with device-side scalars (captured into the body).
int enqueue_iteration(fl_plan_t p, const uint32_t* bits, const double* sigma1, const double* sigma2, double* x,
                      double* work, cudaGraphConditionalHandle h, cudaStream_t s) {
  const int64_t n = p->n;
  double* r = work;
  double* pv = work + 2 * n;
  double* gp = work + 4 * n;
  double* slots = work + 6 * n;
  PcgCtl* ctl = reinterpret_cast<PcgCtl*>(slots + 8);
  Scratch* sc;
  FL_TRY(scratch(&sc));
  const int ksum = RED_SUM;
  int nbg = 0, nbu = 0, nbp = 0;
  bool have_norm = false;
  FL_TRY(op_gram_norm(p, bits, pv, gp, sc->partials, &nbg, &have_norm, s));
  if (!have_norm) FL_TRY(dot_partials(n, pv, gp, sc->partials, &nbg, s));
  FL_TRY(finish_reduce(sc->partials, nbg, 1, &ksum, slots + 2, s));
  FL_TRY(pcg2_update(n, sigma1, sigma2, slots, slots + 2, slots + 3, x, r, pv, gp, sc->partials, &nbu, s));
  FL_TRY(finish_reduce(sc->partials, nbu, 1, &ksum, slots + 1, s));
  k_pcg_control<<<1, 32, 0, s>>>(ctl, slots, h);
  FL_LAUNCH_CHECK();
  FL_TRY(pcg2_pupdate(n, sigma1, sigma2, r, 0.0, pv, sc->partials, &nbp, s, slots + 4, &ctl->done));
  FL_TRY(finish_reduce(sc->partials, nbp, 1, &ksum, slots + 3, s));
  return FL_OK;
}

int pcg_graph(fl_plan_t p, const uint32_t* bits, const double* sigma1, const double* sigma2, double* x,
              double* work, cudaGraphExec_t* out, bool gated = false) {
  Scratch* sc0;
  FL_TRY(scratch(&sc0));
  auto* gs = static_cast<PcgGraphs*>(p->pcg_graphs);
  if (!gs) {
    static std::mutex create_mu;
    std::lock_guard<std::mutex> lock(create_mu);
    if (!p->pcg_graphs) p->pcg_graphs = new PcgGraphs();
    gs = static_cast<PcgGraphs*>(p->pcg_graphs);
  }
  std::lock_guard<std::mutex> lock(gs->mu);
  for (size_t i = 0; i < gs->v.size(); ++i) {
    const PcgGraph& g = gs->v[i];
    if (g.bits == bits && g.sig1 == sigma1 && g.sig2 == sigma2 && g.x == x && g.work == work &&
        g.partials == sc0->partials && g.result == sc0->result && g.gated == gated) {
      PcgGraph hit = g;
      gs->v.erase(gs->v.begin() + (ptrdiff_t)i);
      gs->v.push_back(hit);
      *out = hit.exec;
      return FL_OK;
    }
  }
  if (!gs->capture) FL_CUDA(cudaStreamCreateWithFlags(&gs->capture, cudaStreamNonBlocking));
  if (gs->v.size() >= kPcgGraphCap) {
    destroy_graph(gs->v.front());
    gs->v.erase(gs->v.begin());
  }
  PcgGraph g{bits, sigma1, sigma2, x, work, sc0->partials, sc0->result, gated};
  FL_CUDA(cudaGraphCreate(&g.graph, 0));
  cudaGraphConditionalHandle h;
  // gated: the loop starts closed and k_pcg_gate opens it
  FL_CUDA(cudaGraphConditionalHandleCreate(&h, g.graph, gated ? 0 : 1, cudaGraphCondAssignDefault));
  cudaGraphNode_t gate = nullptr;
  if (gated) {
    Scratch* sc;
    FL_TRY(scratch(&sc));
    PcgCtl* ctl = reinterpret_cast<PcgCtl*>(work + 6 * p->n + 8);
    const double* res = sc->result;
    double* slots = work + 6 * p->n;
    double* dev = sc->result + 32;
    void* args[] = {&ctl, &res, &slots, &dev, &h};
    cudaKernelNodeParams kp = {};
    kp.func = (void*)k_pcg_gate;
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(32);
    kp.kernelParams = args;
    FL_CUDA(cudaGraphAddKernelNode(&gate, g.graph, nullptr, 0, &kp));
  }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  FL_CUDA(cudaGraphAddNode(&node, g.graph, gate ? &gate : nullptr, gate ? 1 : 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  FL_CUDA(cudaStreamBeginCaptureToGraph(gs->capture, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  const int st = enqueue_iteration(p, bits, sigma1, sigma2, x, work, h, gs->capture);
  cudaGraph_t captured = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(gs->capture, &captured);
  if (st != FL_OK || ce != cudaSuccess) {
    cudaGraphDestroy(g.graph);
    return st != FL_OK ? st : fail(FL_E_CUDA, std::string("PCG graph capture: ") + cudaGetErrorString(ce));
  }
  const cudaError_t ie = cudaGraphInstantiate(&g.exec, g.graph, 0);
  if (ie != cudaSuccess) {
    cudaGraphDestroy(g.graph);
    return fail(FL_E_CUDA, std::string("PCG graph instantiate: ") + cudaGetErrorString(ie));
  }
  gs->v.push_back(g);
  *out = g.exec;
  return FL_OK;
}

int pcg_v3_loop(fl_plan_t p, const uint32_t* bits, const double* sigma1, const double* sigma2, double* x,
                double* work, double rho, double abs_tol, double rel_tol, int64_t limit, fl_pcg_result* res,
                cudaStream_t s) {
  const int64_t n = p->n;
  double* slots = work + 6 * n;
  PcgCtl* ctl = reinterpret_cast<PcgCtl*>(slots + 8);
  Scratch* sc;
  FL_TRY(scratch(&sc));
  FL_TRY(check_rho(rho, 0));
  const double norm0 = std::sqrt(rho);
  const double thr = abs_tol + rel_tol * norm0;
  res->norm0 = norm0;
  if (norm0 <= thr || limit <= 0) {
    res->iterations = 0;
    res->converged = norm0 <= thr;
    res->residual_norm = norm0;
    return FL_OK;
  }
  cudaGraphExec_t exec;
  FL_TRY(pcg_graph(p, bits, sigma1, sigma2, x, work, &exec));
  PcgCtl* hc = reinterpret_cast<PcgCtl*>(sc->host);
  *hc = PcgCtl{thr, norm0, 0.0, (long long)limit, 0, 0, 0};
  FL_CUDA(cudaMemcpyAsync(ctl, hc, sizeof(PcgCtl), cudaMemcpyHostToDevice, s));
  FL_CUDA(cudaGraphLaunch(exec, s));
  FL_CUDA(cudaMemcpyAsync(hc, ctl, sizeof(PcgCtl), cudaMemcpyDeviceToHost, s));
  FL_CUDA(cudaStreamSynchronize(s));
  const PcgCtl c = *hc;
  if (c.status == 3) return check_curv(c.bad, c.k);
  if (c.status == 4) return check_rho(c.bad, c.k);
  if (c.status != 1 && c.status != 2) return fail(FL_E_CUDA, "device PCG loop ended without a verdict");
  res->iterations = c.k;
  res->converged = c.status == 1;
  res->residual_norm = c.norm;
  return FL_OK;
}

int pcg_v3(fl_plan_t p, const uint32_t* bits, const double* sigma1, const double* sigma2, const double* rhs,
           double* x, double* work, double abs_tol, double rel_tol, int64_t limit, fl_pcg_result* res,
           cudaStream_t s) {
  const int64_t n = p->n;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  int nb = 0;
  double rho = 0.0;
  FL_TRY(pcg2_init(n, sigma1, sigma2, rhs, x, work, work + 2 * n, sc->partials, &nb, s));
  FL_TRY(pcg_start_fetch(sc, nb, false, work + 6 * n, &rho, nullptr, s));
  return pcg_v3_loop(p, bits, sigma1, sigma2, x, work, rho, abs_tol, rel_tol, limit, res, s);
}


// PCG loop: 3 = one CUDA graph with a device WHILE loop per solve (default),
// 2 = host loop of the same kernels (one sync per iteration).  Set through
// fl_set_pcg_loop (tests compare the two bit for bit).
std::atomic<int> g_pcg_mode{3};
int pcg_mode() { return g_pcg_mode.load(std::memory_order_relaxed); }

int64_t pcg_limit(int64_t n, int64_t max_iters) {
  return max_iters >= 0 ? max_iters : std::min<int64_t>(10 * 2 * n, kPcgIterCap);
}

}  // namespace

namespace fl {
void pcg_graphs_release(fl_plan* p) {
  auto* gs = static_cast<PcgGraphs*>(p->pcg_graphs);
  if (!gs) return;
  for (PcgGraph& g : gs->v) destroy_graph(g);
  if (gs->capture) cudaStreamDestroy(gs->capture);
  delete gs;
  p->pcg_graphs = nullptr;
}
}  // namespace fl

extern "C" {

int64_t fl_pcg_work_doubles(int64_t n) { return 6 * n + 16; }

int fl_set_pcg_loop(int mode) {
  if (mode != 2 && mode != 3) return fail(FL_E_VALUE, "PCG loop mode must be 2 (host) or 3 (device graph)");
  g_pcg_mode.store(mode, std::memory_order_relaxed);
  return FL_OK;
}

int fl_pcg_kkt(fl_plan_t p, const uint32_t* bits, const double* sigma1, const double* sigma2,
               const double* rhs, double* x, double* work, double abs_tol, double rel_tol,
               int64_t max_iters, fl_pcg_result* res, double* history, int64_t max_history,
               fl_stream_t stream) {
  if (!p || !bits || !sigma1 || !sigma2 || !rhs || !x || !work || !res)
    return fail(FL_E_VALUE, "null argument");
  if (abs_tol < 0 || rel_tol < 0) return fail(FL_E_VALUE, "tolerances must be nonnegative");
  if (abs_tol == 0 && rel_tol == 0) return fail(FL_E_VALUE, "abs_tol and rel_tol cannot both be zero");
  const int64_t limit = pcg_limit(p->n, max_iters);
  const int mode = pcg_mode();
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 3 && !(history && max_history > 0))
    return pcg_v3(p, bits, sigma1, sigma2, rhs, x, work, abs_tol, rel_tol, limit, res, s);
  return pcg_v2(p, bits, sigma1, sigma2, rhs, x, work, abs_tol, rel_tol, limit, res, history, max_history, s);
}

int fl_ipm_newton_pcg(fl_plan_t p, const uint32_t* bits, const fl_state* st, const double* g, double lam,
                      double mu, double* sigma1, double* sigma2, double* x, double* work, double abs_tol,
                      double rel_tol, int64_t max_iters, fl_pcg_result* res, fl_stream_t stream) {
  if (!p || !bits || !st || !g || !sigma1 || !sigma2 || !x || !work || !res)
    return fail(FL_E_VALUE, "null argument");
  if (abs_tol < 0 || rel_tol < 0) return fail(FL_E_VALUE, "tolerances must be nonnegative");
  if (abs_tol == 0 && rel_tol == 0) return fail(FL_E_VALUE, "abs_tol and rel_tol cannot both be zero");
  const int64_t n = p->n;
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  int nb = 0;
  double rho = 0.0, flag = 0.0;
  FL_TRY(newton_setup(n, st, g, lam, mu, sigma1, sigma2, x, work, work + 2 * n, sc->partials, &nb, s));
  FL_TRY(pcg_start_fetch(sc, nb, true, work + 6 * n, &rho, &flag, s));
  if (flag != 0.0) return fail(FL_E_INTERIOR, "slacks and multipliers must be strictly positive and finite");
  const int64_t limit = pcg_limit(n, max_iters);
  if (pcg_mode() == 3)
    return pcg_v3_loop(p, bits, sigma1, sigma2, x, work, rho, abs_tol, rel_tol, limit, res, s);
  return pcg_v2_loop(p, bits, sigma1, sigma2, x, work, rho, abs_tol, rel_tol, limit, res, nullptr, 0, s);
}


// One IPM step with a single host sync before the loop's convergence check
// (ipm.py:364-394): newton_setup + PCG as fl_ipm_newton_pcg, then ratios,
// device step lengths, the gated state update and the interior flag
// (ipm_step_device), and ONE asynchronous copy of the step verdict to
// ``host_out`` (13 doubles, pinned): [0..3] ratio minima, [4] alpha_p,
// [5] alpha_d, [6] skipped, [7] interior flag, [8] PCG status (1 converged,
// 2 iteration cap, 3 curvature breakdown, 4 r'P^{-1}r breakdown), [9] PCG
// iterations, [10] residual norm, [11] offending value, [12] initial norm.
// Valid after the caller's next stream sync (fl_ipm_assess).
int fl_ipm_newton_step(fl_plan_t p, const uint32_t* bits, const fl_state* st, const double* g, double lam,
                       double mu, double tau, double* sigma1, double* sigma2, double* x, double* work,
                       double abs_tol, double rel_tol, int64_t max_iters, double* host_out, fl_stream_t stream) {
  if (!p || !bits || !st || !g || !sigma1 || !sigma2 || !x || !work || !host_out)
    return fail(FL_E_VALUE, "null argument");
  if (abs_tol < 0 || rel_tol < 0) return fail(FL_E_VALUE, "tolerances must be nonnegative");
  if (abs_tol == 0 && rel_tol == 0) return fail(FL_E_VALUE, "abs_tol and rel_tol cannot both be zero");
  const int64_t n = p->n;
  cudaStream_t s = (cudaStream_t)stream;
  Scratch* sc;
  FL_TRY(scratch(&sc));
  int nb = 0;
  double rho = 0.0, flag = 0.0;
  FL_TRY(newton_setup(n, st, g, lam, mu, sigma1, sigma2, x, work, work + 2 * n, sc->partials, &nb, s));
  const int64_t limit = pcg_limit(n, max_iters);
  double* slots = work + 6 * n;
  PcgCtl* ctl = reinterpret_cast<PcgCtl*>(slots + 8);
  PcgCtl* hc = reinterpret_cast<PcgCtl*>(sc->host);
  double* dev = sc->result + 32;
  if (pcg_mode() == 3) {
    // no sync at all: the start check runs in the graph's gate kernel
    const int kinds[3] = {RED_SUM, RED_SUM, RED_MAX};
    FL_TRY(finish_reduce(sc->partials, nb, 3, kinds, sc->result, s));
    cudaGraphExec_t exec;
    FL_TRY(pcg_graph(p, bits, sigma1, sigma2, x, work, &exec, true));
    *hc = PcgCtl{0.0, 0.0, 0.0, (long long)limit, 0, 0, 0, abs_tol, rel_tol};
    FL_CUDA(cudaMemcpyAsync(ctl, hc, sizeof(PcgCtl), cudaMemcpyHostToDevice, s));
    FL_CUDA(cudaGraphLaunch(exec, s));
    FL_TRY(ipm_step_device(n, st, sigma1, sigma2, mu, tau, x, x + n, &ctl->status, dev, s));
    k_step_pack<<<1, 32, 0, s>>>(ctl, -1.0, dev);
    FL_LAUNCH_CHECK();
    FL_CUDA(cudaMemcpyAsync(host_out, dev, 13 * sizeof(double), cudaMemcpyDeviceToHost, s));
    return FL_OK;
  }
  FL_TRY(pcg_start_fetch(sc, nb, true, work + 6 * n, &rho, &flag, s));
  if (flag != 0.0) return fail(FL_E_INTERIOR, "slacks and multipliers must be strictly positive and finite");
  FL_TRY(check_rho(rho, 0));
  const double norm0 = std::sqrt(rho);
  const double thr = abs_tol + rel_tol * norm0;
  if (norm0 <= thr || limit <= 0) {
    *hc = PcgCtl{thr, norm0, 0.0, (long long)limit, 0, norm0 <= thr ? 1 : 2, 1};
    FL_CUDA(cudaMemcpyAsync(ctl, hc, sizeof(PcgCtl), cudaMemcpyHostToDevice, s));
  } else {
    fl_pcg_result r{};
    FL_TRY(pcg_v2_loop(p, bits, sigma1, sigma2, x, work, rho, abs_tol, rel_tol, limit, &r, nullptr, 0, s));
    *hc = PcgCtl{thr, r.residual_norm, 0.0, (long long)limit, (long long)r.iterations, r.converged ? 1 : 2, 1};
    FL_CUDA(cudaMemcpyAsync(ctl, hc, sizeof(PcgCtl), cudaMemcpyHostToDevice, s));
  }
  FL_TRY(ipm_step_device(n, st, sigma1, sigma2, mu, tau, x, x + n, &ctl->status, dev, s));
  k_step_pack<<<1, 32, 0, s>>>(ctl, norm0, dev);
  FL_LAUNCH_CHECK();
  FL_CUDA(cudaMemcpyAsync(host_out, dev, 13 * sizeof(double), cudaMemcpyDeviceToHost, s));
  return FL_OK;
}

}  // extern "C"
