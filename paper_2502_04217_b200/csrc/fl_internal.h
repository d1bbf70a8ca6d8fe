// Internal (C++) interfaces shared between the translation units of
// libfftlasso_b200.  Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "fl_fft.cuh"
#include "fftlasso_b200.h"

// Four-step decomposition of an axis too long for one CTA's shared memory.
struct LongAxis {
  bool on = false;
  int m1 = 0, m2 = 0;
  fl::AxisPlan p1, p2;
  double2* scratch = nullptr;  // G * m complex
};

struct fl_plan {
  int ndim = 0;
  int64_t dims[3] = {1, 1, 1};
  int64_t n = 0;
  int device = 0;
  fl::AxisPlan axis[3];
  LongAxis lng[3];
  bool planned[3] = {true, true, true};  // false: batch extent of a slab plan
  std::vector<void*> owned;  // device allocations (twiddle tables)
  void* pcg_graphs = nullptr;  // cached device-looped PCG graphs (fl_pcg.cu)
};

namespace fl {

constexpr int kMaxDevices = 16;  // per-device caches (scratch, kernel attributes)

enum PassKind : int { K_SYNTH = 0, K_ANALYZE = 1, K_GRAM = 2, K_RESID = 3 };

struct KktEpi {
  const double* pb = nullptr;   // d_beta
  const double* pz = nullptr;   // d_z
  const double* sig1 = nullptr;
  const double* sig2 = nullptr;
  double* bottom = nullptr;     // optional
  double* partials = nullptr;   // non-null: per-block d.Kd partials
};

// One axis pass over the grid; returns grid size used (for partial slots) in *nblocks.
int run_pass(const fl_plan* p, int axis, int kind, const double* in, double* out,
             const uint32_t* bits, const double* bhat, const KktEpi* epi, int* nblocks,
             cudaStream_t s);

int run_pass_n(const fl_plan* p, int axis, int kind, const double* in, double* out,
               const uint32_t* bits, const double* bhat, const KktEpi* epi, int* nblocks,
               double* nrm_partials, cudaStream_t s);
int op_gram_norm(const fl_plan* p, const uint32_t* bits, const double* in, double* out,
                 double* nrm_partials, int* nblocks, bool* have_norm, cudaStream_t s);

struct PassArgs;
int long_factor(int m, int* m1, int* m2);
int run_long(const fl_plan* p, int axis, int kind, const PassArgs& A, bool strided, const KktEpi* epi,
             int* nblocks, cudaStream_t s);

// Whole-operator sequences (fl_pass.cu)
int op_synthesize(const fl_plan* p, const double* in, double* out, cudaStream_t s);
int op_analyze(const fl_plan* p, const double* in, double* out, cudaStream_t s);
// gram (resid=false) or A^T Z (bhat - A in) (resid=true); optional KKT epilogue on the last pass.
int op_gram(const fl_plan* p, const uint32_t* bits, const double* bhat, bool resid,
            const double* in, double* out, const KktEpi* epi, int* nblocks, cudaStream_t s);

// KKT apply in the axis-0-last order with the epilogue fused (fl_pass.cu)
bool kkt_order_b(const fl_plan* p);

// Elementwise KKT epilogue on a gram output (fl_vec.cu); n even.
int kkt_epilogue(int64_t n, double* g, const double* pb, const double* pz, const double* sig1,
                 const double* sig2, double* bottom, double* partials, int* nblocks, cudaStream_t s);

// PCG kernels (fl_vec.cu)
// restructured PCG: curvature = ||Z A p_beta||^2 (fused gram pass) + diagonal form
int pcg2_init(int64_t n, const double* sig1, const double* sig2, const double* rhs, double* x, double* r,
              double* p, double* partials, int* nblocks, cudaStream_t s);
int ipm_step_device(int64_t n, const fl_state* st, const double* sigma1, const double* sigma2, double mu,
                    double tau, const double* d_beta, const double* d_z, const int* pcg_status, double* dev,
                    cudaStream_t s);
int pcg2_update(int64_t n, const double* sig1, const double* sig2, const double* rho, const double* curv_g,
                const double* curv_d, double* x, double* r, const double* p, const double* gp,
                double* partials, int* nblocks, cudaStream_t s);
// beta_dev (optional) overrides beta on the device; done (optional) makes the
// kernel a no-op once the device-looped PCG has stopped.
int pcg2_pupdate(int64_t n, const double* sig1, const double* sig2, const double* r, double beta, double* p,
                 double* partials, int* nblocks, cudaStream_t s, const double* beta_dev = nullptr,
                 const int* done = nullptr);
// Release the plan's cached PCG graphs (fl_plan_destroy).
void pcg_graphs_release(fl_plan* p);
int dot_partials(int64_t n, const double* a, const double* b, double* partials, int* nblocks, cudaStream_t s);
// Fused barrier diagonals + condensed RHS + PCG start (rows: rho, diag curvature, interior flag).
int newton_setup(int64_t n, const fl_state* st, const double* g, double lam, double mu, double* sig1,
                 double* sig2, double* x, double* r, double* p, double* partials, int* nblocks, cudaStream_t s);

}  // namespace fl
