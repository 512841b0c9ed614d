// emrkc_capi.cpp — host side of libemrkc_b200.so: the C ABI of
// include/emrkc.h. Planning, RKC coefficients, device buffers, the step /
// run loops, the device power iteration and z-slab groups.
//
// The host numerics restate the reference's scalar routines (get_stages,
// rkc_coeffs, resting_state, P/src/cheb.cpp:8-69, P/src/ionic.cpp:14-116)
// in the same evaluation order so that s, m, eta and every coefficient are
// bit-identical; all per-node work runs in kernels.cu. There is no CPU
// fallback: without a device every compute call fails with EMRKC_ECUDA.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <array>
#include <random>
#include <string>
#include <vector>

#include "../../include/emrkc.h"
#include "kernels.h"

using emrkc_k::Geom;
using emrkc_k::Halo;
using emrkc_k::kNoEvent;
using emrkc_k::StageArgs;

namespace {

thread_local std::string g_global_err;

int set_global(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_global_err = buf;
  return code;
}

// ---------------------------------------------------------------------------
// Host numerics (restated from the reference, same operation order)
// ---------------------------------------------------------------------------
struct Cheb {
  double value, derivative;
};

Cheb cheb_T(int degree, double x) {  // P/src/cheb.cpp:8-23
  double tm1 = 1.0, dm1 = 0.0;
  if (degree == 0) return {tm1, dm1};
  double t = x, d = 1.0;
  for (int j = 2; j <= degree; ++j) {
    const double tj = 2.0 * x * t - tm1;
    const double dj = 2.0 * t + 2.0 * x * d - dm1;
    tm1 = t;
    dm1 = d;
    t = tj;
    d = dj;
  }
  return {t, d};
}

struct Coeffs {
  int s = 0;
  double omega0 = 0, omega1 = 0;
  std::vector<double> b, mu, nu, kappa, c;
};

int stages(double dt, double rho, double eps, int32_t* s, double* ell,
           double* beta) {  // P/src/cheb.cpp:25-39
  if (!std::isfinite(dt) || !std::isfinite(rho) || !std::isfinite(eps))
    return set_global(EMRKC_EINVAL, "get_stages: non-finite input");
  if (dt <= 0.0) return set_global(EMRKC_EINVAL, "get_stages: dt must be > 0");
  if (rho < 0.0) return set_global(EMRKC_EINVAL, "get_stages: rho must be >= 0");
  if (eps < 0.0 || eps >= 1.5)
    return set_global(EMRKC_EINVAL, "get_stages: damping must be in [0, 1.5)");
  const double b = 2.0 - 4.0 * eps / 3.0;
  const double q = std::ceil(std::sqrt(dt * rho / b));
  if (!(q < 1e6))
    return set_global(EMRKC_EINVAL, "get_stages: stage count overflow");
  const int si = std::max(1, static_cast<int>(q));
  *s = si;
  *ell = b * static_cast<double>(si) * si;
  *beta = b;
  return EMRKC_OK;
}

int coeffs(int s, double eps, Coeffs* k) {  // P/src/cheb.cpp:41-69
  if (s < 1) return set_global(EMRKC_EINVAL, "rkc_coeffs: s must be >= 1");
  k->s = s;
  k->omega0 = 1.0 + eps / (static_cast<double>(s) * s);
  const Cheb ts = cheb_T(s, k->omega0);
  k->omega1 = ts.value / ts.derivative;
  k->b.assign(s + 1, 0.0);
  for (int j = 0; j <= s; ++j) k->b[j] = 1.0 / cheb_T(j, k->omega0).value;
  k->mu.assign(s + 1, 0.0);
  k->nu.assign(s + 1, 0.0);
  k->kappa.assign(s + 1, 0.0);
  k->c.assign(s + 1, 0.0);
  k->mu[1] = k->omega1 / k->omega0;
  k->c[1] = k->mu[1];
  for (int j = 2; j <= s; ++j) {
    k->mu[j] = 2.0 * k->omega1 * k->b[j] / k->b[j - 1];
    k->nu[j] = 2.0 * k->omega0 * k->b[j] / k->b[j - 1];
    k->kappa[j] = -k->b[j] / k->b[j - 2];
    k->c[j] = k->nu[j] * k->c[j - 1] + k->kappa[j] * k->c[j - 2] + k->mu[j];
  }
  return EMRKC_OK;
}

// HH on the host, for the resting state only (P/src/ionic.cpp:14-116).
double lin_exp_ratio(double x, double k) {
  const double u = x / k;
  if (std::abs(u) < 1e-4) return k * (1.0 + u * (0.5 + u / 12.0));
  return x / (1.0 - std::exp(-u));
}
// HH rates alpha_g, beta_g (P/src/ionic.cpp:98-109)
void hh_rates(double V, double* a, double* b) {
  a[0] = 0.1 * lin_exp_ratio(V + 40.0, 10.0);
  b[0] = 4.0 * std::exp(-(V + 65.0) / 18.0);
  a[1] = 0.07 * std::exp(-(V + 65.0) / 20.0);
  b[1] = 1.0 / (1.0 + std::exp(-(V + 35.0) / 10.0));
  a[2] = 0.01 * lin_exp_ratio(V + 55.0, 10.0);
  b[2] = 0.125 * std::exp(-(V + 65.0) / 80.0);
}
void hh_gate_coeffs(double V, double* lam, double* zinf) {
  double a[3], b[3];
  hh_rates(V, a, b);
  for (int g = 0; g < 3; ++g) {
    lam[g] = -(a[g] + b[g]);
    zinf[g] = a[g] / (a[g] + b[g]);
  }
}
double hh_current(double V, const double* z) {
  const double m = z[0], h = z[1], n = z[2];
  return 1.2 * m * m * m * h * (V - 50.0) + 0.36 * n * n * n * n * (V - -77.0) +
         0.003 * (V - -54.387);
}

// Per-step plan: plan_step (P/src/multirate.cpp:129-135) + coefficients.
// Stepping methods of the device path (Method, P/include/mrkc/config.hpp:17).
enum { kMethodEmrkc = 0, kMethodEmrkcProgressive = 1, kMethodExexRl = 2, kMethodMrkc = 3 };

// exp-part evaluations per step (EvalCounters::n_exp_steps): none in mRKC
inline int exp_per_step(int method, int s) { return method == kMethodMrkc ? 0 : s; }

struct Plan {
  double dt = -1, eps = -1, rho_F = -1, rho_S = -1;
  int method = -1;
  int s = 0, m = 0;
  // gate rows of the averaged force: (u_m - z)/eta = gate_c (y_E - z)/eta.
  // standard: u_m = y_E (the inner iterate starts at y_E and f vanishes on
  // gate rows); progressive: the inner iteration starts at y with the
  // constant forcing (y_E - y)/eta on gate rows (P/src/multirate.cpp:106-115),
  // so u_m - y = c_m (y_E - y) with the inner RKC's c_m (= 1 up to rounding).
  double gate_c = 1.0;
  int exex = 0;
  double eta = 0, ell_s = 0, ell_m = 0, beta = 0;
  Coeffs outer, inner;
  std::vector<double> in_mueta;  // mu'_k * eta (rkc_iteration's k.mu[j]*dt)
  std::vector<double> mudt;      // mu_j * dt
};

int make_plan(double dt, double rho_F, double rho_S, double eps, Plan* p,
              int method = kMethodEmrkc) {
  if (!(dt > 0.0)) return set_global(EMRKC_EINVAL, "emrkc_step: dt must be > 0");
  p->method = method;
  p->gate_c = 1.0;
  p->exex = 0;
  if (method == kMethodExexRl) {
    // exex_rl_step (P/src/baselines.cpp:192-210) as the one-stage kernel:
    // gates y + expm1(dt Lambda)(y - y_inf), V + dt (f_F(V) + v_reaction at
    // the new gates) = the m = s = 1 node update with eta = dt, mu_1 = 1,
    // mu'_1 = 1 (so cG = 1 and cV = dt).
    p->s = p->m = 1;
    p->eta = dt;
    p->ell_s = p->ell_m = p->beta = 0.0;
    int rc;
    if ((rc = coeffs(1, 0.05, &p->outer))) return rc;
    if ((rc = coeffs(1, 0.05, &p->inner))) return rc;
    p->in_mueta.assign(2, 0.0);
    p->in_mueta[1] = dt;
    p->mudt.assign(2, 0.0);
    p->mudt[1] = dt;
    p->exex = 1;
    p->dt = dt;
    p->eps = eps;
    p->rho_F = rho_F;
    p->rho_S = rho_S;
    return EMRKC_OK;
  }
  int rc = stages(dt, rho_S, eps, &p->s, &p->ell_s, &p->beta);
  if (rc) return rc;
  p->eta = 2.0 * dt / p->ell_s;
  rc = stages(p->eta, rho_F, eps, &p->m, &p->ell_m, &p->beta);
  if (rc) return rc;
  if ((rc = coeffs(p->s, eps, &p->outer))) return rc;
  if ((rc = coeffs(p->m, eps, &p->inner))) return rc;
  p->in_mueta.assign(p->m + 1, 0.0);
  for (int k = 1; k <= p->m; ++k) p->in_mueta[k] = p->inner.mu[k] * p->eta;
  p->mudt.assign(p->s + 1, 0.0);
  for (int j = 1; j <= p->s; ++j) p->mudt[j] = p->outer.mu[j] * dt;
  if (method == kMethodEmrkcProgressive) p->gate_c = p->inner.c[p->m];
  p->dt = dt;
  p->eps = eps;
  p->rho_F = rho_F;
  p->rho_S = rho_S;
  return EMRKC_OK;
}

int64_t nodes_of(const emrkc_problem* p) {
  int64_t nn = 1;
  for (int a = 0; a < p->dim; ++a) nn *= p->n[a];
  return nn;
}

// SoA fields of a state: V, 3 HH gates, the aux variables of
// EMRKC_MODEL_HH_AUX (include/emrkc.h)
int fields_of(const emrkc_problem* p) {
  return 4 + (p->model == EMRKC_MODEL_HH_AUX ? p->n_aux : 0);
}
double aux_s1(int a) { return 0.01 * static_cast<double>(a % 3); }
double aux_s0(int a) { return 0.5 + 0.1 * static_cast<double>(a % 4); }

int validate(const emrkc_problem* p) {
  if (!p) return set_global(EMRKC_EINVAL, "null problem");
  if (p->dim < 1 || p->dim > 3)
    return set_global(EMRKC_EINVAL, "grid: dim must be 1, 2, or 3");
  if (p->model != EMRKC_MODEL_HH && p->model != EMRKC_MODEL_HH_AUX)
    return set_global(EMRKC_EINVAL, "unknown ionic model %d", p->model);
  if (p->model == EMRKC_MODEL_HH_AUX && (p->n_aux < 1 || p->n_aux > EMRKC_MAX_AUX))
    return set_global(EMRKC_EINVAL, "hh_aux: n_aux must be in [1, %d]", EMRKC_MAX_AUX);
  for (int a = 0; a < p->dim; ++a) {
    if (p->n[a] < 2 || !(p->dx[a] > 0.0))
      return set_global(EMRKC_EINVAL, "grid: extent and dx must be positive");
    if (p->n[a] > (1 << 30))
      return set_global(EMRKC_EINVAL, "grid: axis too long");
  }
  for (int a = p->dim; a < 3; ++a)
    if (p->n[a] != 1) return set_global(EMRKC_EINVAL, "grid: unused axes need n = 1");
  if (!(p->chi > 0.0) || !(p->C_m > 0.0))
    return set_global(EMRKC_EINVAL, "conductivity: chi and C_m must be > 0");
  return EMRKC_OK;
}

// Stimulus node range of one axis: the reference's per-node test
// x = i*dx against [lo - 1e-12, hi + 1e-12] (P/src/monodomain.cpp:151-158)
// evaluated for every index; the accepted set is an interval.
void stim_range(const emrkc_problem* p, int a, int* lo, int* hi) {
  *lo = 1;
  *hi = 0;
  bool any = false;
  for (int64_t i = 0; i < p->n[a]; ++i) {
    const double x = static_cast<double>(i) * p->dx[a];
    if (!(x < p->stim_lo[a] - 1e-12 || x > p->stim_hi[a] + 1e-12)) {
      if (!any) *lo = static_cast<int>(i);
      *hi = static_cast<int>(i);
      any = true;
    }
  }
}

double stim_rate_at(const emrkc_problem* p, double t) {
  // stimulus_rate's time/amplitude part (P/src/monodomain.cpp:152,157) and
  // StimulusProtocol::active_at (P/include/mrkc/monodomain.hpp:71)
  if (p->stim_chi_amplitude == 0.0 || !(t >= p->stim_t0 && t <= p->stim_t1))
    return 0.0;
  return p->stim_chi_amplitude / (p->chi * p->C_m);
}

}  // namespace

// ---------------------------------------------------------------------------
// Handle
// ---------------------------------------------------------------------------
struct emrkc_handle {
  emrkc_problem p{};
  int device = 0;
  cudaStream_t stream = nullptr;
  Geom geom{};
  int64_t nn = 0, len = 0;
  int64_t z_begin = 0, z_end = 0;
  bool partitioned = false;
  double* buf[4] = {nullptr, nullptr, nullptr, nullptr};
  int nbuf = 0;
  int cur = 0;
  bool has_state = false;
  // m >= 2 scratch
  double* fs = nullptr;
  double* ye = nullptr;
  double* u[4] = {nullptr, nullptr, nullptr, nullptr};
  // ghost planes [side: 0 below, 1 above][slot], carved from one arena that
  // also holds the arrival counters of the cross-process protocol
  double* ghost[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  // 3-D slabs: d_1 ghosts of the wide halo [side][outer-stage parity],
  // kTbMaxK planes each (k_vin_tb on slabs)
  double* dghost[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  int64_t min_depth = 0;  // smallest slab depth of the partition (0: unknown)
  long long kstage = 0;   // wide-halo outer stages run (d_1 ghost parity)
  void* arena = nullptr;
  size_t arena_bytes = 0;
  unsigned long long* cnt = nullptr;         // [2]: arrivals into ghost[0] / ghost[1]
  emrkc_handle* nbr[2] = {nullptr, nullptr};  // in-process neighbours
  // cross-process (or in-process lockstep) neighbours: their arena pointers
  struct {
    bool linked = false;
    bool ipc = false;           // opened with cudaIpcOpenMemHandle
    void* arena = nullptr;
    double* ghost[2] = {nullptr, nullptr};  // their ghost[1-side][slot]
    double* dghost[2] = {nullptr, nullptr}; // their dghost[1-side][parity]
    unsigned long long* cnt = nullptr;      // their cnt[1-side]
  } peer[2];
  unsigned long long recv[2] = {0, 0};  // arrivals expected so far per side
  double* ckpt = nullptr;               // dist_run input state, for replay
  emrkc_level_hook level_hook = nullptr;  // testing aid (emrkc_set_level_hook)
  void* level_ctx = nullptr;
  double* res_v = nullptr;              // resident runs: V ping-pong [2][nn]
  double* res_stim = nullptr;           // resident runs: stimulus rate per step
  int64_t res_stim_n = 0;
  long long level = 0;
  // device scalars
  unsigned long long* d_event = nullptr;
  unsigned long long* d_slots = nullptr;
  const unsigned long long* slot_init = nullptr;  // run loops: slot of the initial state's gate range
  size_t slots_cap = 0;
  double* d_coef = nullptr;  // in_mueta | in_nu | in_kappa (3*(m+1))
  size_t coef_cap = 0;
  double* d_red = nullptr;   // reduction partials + scalar
  double* d_rel = nullptr;   // rel_l2_error partials
  double* d_tmp = nullptr;   // one node field (host reference upload)
  Plan plan;
  bool plan_uploaded = false;
  int fast = 1;
  int pipe = 1;
  int method = 0;  // kMethod* of the next plan (set by the API entry point)
  int tb = 1;      // temporally blocked inner stages 2..m in one pass (k_vin_tb,
                   // 3 <= m <= 5; EMRKC_TB=0: one kernel per stage)
  int pair = 1;    // pair-per-thread node kernel on 3-D whole grids (EMRKC_PAIR=0: k_node_tma)
  int xstep = 0;   // cross-step fusion of the s = 1, m = 2 step in run loops (EMRKC_XSTEP=1)
  int stiff = 1;   // mRKC stiff-gate split: gates in the fast part (bit 0 = m)
  double* mr_u[3] = {nullptr, nullptr, nullptr};  // mRKC inner stages (4 blocks each)
  double* mr_fs = nullptr;                        // mRKC frozen slow term
  double* cg_v = nullptr;   // IMEX-RL CG vectors b, x, r, z, p, q (6 n_nodes)
  double* cg_part = nullptr;  // CG partial sums (3 * power_blocks())
  emrkc_k::CgScalars* cg_s = nullptr;   // device scalars
  emrkc_k::CgScalars* cg_h = nullptr;   // pinned host copy
  int* guard_d = nullptr;
  int zr_lo = -1, zr_hi = -1;  // node-kernel plane range override (< 0: all)
  // z-pipelined step (EMRKC_ZPIPE): inner-stage chunks on a second stream,
  // each chunk behind the node-kernel chunk it needs
  int zpipe = 0;                     // EMRKC_ZPIPE chunks (0: off; measured slower)
  cudaStream_t s_aux = nullptr;      // stream of the inner-stage chunks
  cudaStream_t ls = nullptr;         // launch_level's stream (null: stream)
  std::vector<cudaEvent_t> zp_ev;    // node chunk c done
  cudaEvent_t zp_join = nullptr;     // inner chunks of the step done
  // fused s = 1, m = 2 step (k_fused2): tile plan, exchange ring, flags
  int fused = 0;                    // EMRKC_FUSED=1: the fused s = 1, m = 2 pass (slower
                                    // on B200 than the two-kernel step)
  int fu_ntx = 0, fu_nty = 0, fu_nzc = 0;  // 0: not planned / not possible
  bool fu_planned = false;
  // slab power iteration driven across processes (emrkc_slab_power_*)
  double* sp_v[2] = {nullptr, nullptr};
  double* sp_fy = nullptr;
  int sp_code = -1, sp_a = 0;
  double* fu_xch = nullptr;
  unsigned long long* fu_flags = nullptr;
  unsigned long long fu_epoch = 0;
  // pipelined host step (emrkc_step_host): copy streams and chunk events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  unsigned long long* h_event = nullptr;  // pinned copy of the abort word
  std::vector<cudaEvent_t> ev_in, ev_k;
  // TMA descriptors (pipe == 3), encoded on first use per (pointer, kind)
  struct TmaEntry {
    const void* ptr;
    int kind;
    CUtensorMap map;
  };
  std::vector<TmaEntry> tmaps;
  int zc = 1;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::string err;
};

struct emrkc_group {
  std::vector<emrkc_handle*> hs;
};

namespace {

int set_err(emrkc_handle* h, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  g_global_err = buf;
  return code;
}

#define CK(h, call)                                                          \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess)                                                   \
      return set_err((h), EMRKC_ECUDA, "%s: %s (%s:%d)", #call,              \
                     cudaGetErrorString(e_), __FILE__, __LINE__);            \
  } while (0)

cudaStream_t lstream(const emrkc_handle* h) { return h->ls ? h->ls : h->stream; }

int use_device(emrkc_handle* h) {
  CK(h, cudaSetDevice(h->device));
  return EMRKC_OK;
}

// Ghost arena of a partitioned handle (both ends of a link compute the same
// layout): V ghost planes [side][slot] (4 planes), then for 3-D the d_1 ghosts
// of the wide halo [side][parity][kTbMaxK planes], then the two arrival
// counters.
size_t arena_planes(int dim) { return 4 + (dim == 3 ? 4 * emrkc_k::kTbMaxK : 0); }
double* dghost_at(double* base, size_t pl, int side, int par) {
  return base + (4 + static_cast<size_t>(2 * side + par) * emrkc_k::kTbMaxK) * pl;
}

// The fast ionic path's V window for this eta (fast_math.cuh) as centre and
// radius: |V - vmid| <= vrad (empty window: vrad < 0, never fast).
// Lower end: the smallest V >= -400 with eta * (alpha_g + beta_g) <= 580 for
// every gate, solved on the reference's own rates (hh_rates) by bisection
// where the sum falls with V (beta_m, beta_n below rest), then checked by a
// scan of [vlo, min(vhi, 200)] against 600 (the table exp's exponent
// insertion wraps near -708). Upper end: kernels.h fast_vhi (alpha_m ~
// 0.1 (V + 40) dominates there).
void fast_window_solve(double eta, double* vmid, double* vrad) {
  auto worst = [eta](double V) {
    double a[3], b[3];
    hh_rates(V, a, b);
    return eta * std::max({a[0] + b[0], a[1] + b[1], a[2] + b[2]});
  };
  const double hi = emrkc_k::fast_vhi(eta);
  double lo = -400.0;
  if (!(eta > 0.0) || worst(-50.0) > 580.0) {
    *vmid = 0.0;
    *vrad = -1.0;
    return;
  }
  if (worst(lo) > 580.0) {
    double a = -400.0, b = -50.0;  // worst(a) > 580 >= worst(b)
    for (int it = 0; it < 80; ++it) {
      const double c = 0.5 * (a + b);
      (worst(c) > 580.0 ? a : b) = c;
    }
    lo = b;
  }
  for (double V = lo, top = std::min(hi, 200.0); V <= top; V += 0.01)
    if (worst(V) > 600.0) {
      *vmid = 0.0;
      *vrad = -1.0;
      return;
    }
  *vmid = 0.5 * (lo + hi);
  *vrad = 0.5 * (hi - lo);
}
// Per launch: the last eta's window is kept per host thread (a run has one
// eta; the scan above costs ~1 ms).
void fast_window(double eta, double* vmid, double* vrad) {
  thread_local double k_eta = -1.0, k_mid = 0.0, k_rad = -1.0;
  if (eta != k_eta) {
    fast_window_solve(eta, &k_mid, &k_rad);
    k_eta = eta;
  }
  *vmid = k_mid;
  *vrad = k_rad;
}

int ensure_buffers(emrkc_handle* h, int nb) {
  for (int i = h->nbuf; i < nb; ++i)
    CK(h, cudaMalloc(&h->buf[i], sizeof(double) * h->len));
  if (nb > h->nbuf) h->nbuf = nb;
  return EMRKC_OK;
}

int ensure_inner(emrkc_handle* h) {
  if (h->fs) return EMRKC_OK;
  CK(h, cudaMalloc(&h->fs, sizeof(double) * h->nn));
  CK(h, cudaMalloc(&h->ye, sizeof(double) * 3 * h->nn));
  for (int k = 0; k < 4; ++k) CK(h, cudaMalloc(&h->u[k], sizeof(double) * h->nn));
  return EMRKC_OK;
}

int ensure_slots(emrkc_handle* h, size_t nsteps) {
  const size_t need = 2 * (nsteps + 1);
  if (need <= h->slots_cap) return EMRKC_OK;
  if (h->d_slots) cudaFree(h->d_slots);
  CK(h, cudaMalloc(&h->d_slots, sizeof(unsigned long long) * need));
  h->slots_cap = need;
  return EMRKC_OK;
}

int upload_plan(emrkc_handle* h, double dt, double rho_F, double rho_S,
                double eps) {
  Plan& pl = h->plan;
  if (pl.dt == dt && pl.rho_F == rho_F && pl.rho_S == rho_S && pl.eps == eps &&
      pl.method == h->method && h->plan_uploaded)
    return EMRKC_OK;
  if ((h->method == kMethodEmrkcProgressive || h->method == kMethodExexRl) && !h->fast)
    return set_err(h, EMRKC_EINVAL,
                   "the progressive variant and EXEX-RL run on the fast kernels (EMRKC_FAST=1)");
  if (h->geom.naux > 0 &&
      (h->method == kMethodExexRl || h->method == kMethodMrkc || !h->fast || h->pipe != 3 ||
       h->geom.dim < 2))
    return set_err(h, EMRKC_EINVAL,
                   "hh_aux (the synthetic width stand-in) runs emRKC (standard / progressive) "
                   "on the TMA kernels of 2-D / 3-D grids only");
  int rc = make_plan(dt, rho_F, rho_S, eps, &pl, h->method);
  if (rc) return set_err(h, rc, "%s", g_global_err.c_str());
  const size_t need = 3 * (pl.m + 1);
  if (need > h->coef_cap) {
    if (h->d_coef) cudaFree(h->d_coef);
    CK(h, cudaMalloc(&h->d_coef, sizeof(double) * need));
    h->coef_cap = need;
  }
  std::vector<double> host(need, 0.0);
  for (int k = 0; k <= pl.m; ++k) {
    host[k] = pl.in_mueta[k];
    host[(pl.m + 1) + k] = pl.inner.nu[k];
    host[2 * (pl.m + 1) + k] = pl.inner.kappa[k];
  }
  CK(h, cudaMemcpy(h->d_coef, host.data(), sizeof(double) * need,
                   cudaMemcpyHostToDevice));
  const int nb = pl.s == 1 ? 2 : (pl.s == 2 ? 3 : 4);
  if ((rc = ensure_buffers(h, nb))) return rc;
  if (pl.m >= 2 && (rc = ensure_inner(h))) return rc;
  h->plan_uploaded = true;
  return EMRKC_OK;
}

// Ghost planes consumed at stencil level L (slot L%2), and where this
// handle's produced plane goes (the neighbour's slot (L+1)%2).
Halo halo_at(const emrkc_handle* h, long long L) {
  Halo x{};
  const int rs = static_cast<int>(L & 1), ws = static_cast<int>((L + 1) & 1);
  if (h->nbr[0]) {
    x.lo = h->ghost[0][rs];
    x.put_lo = h->nbr[0]->ghost[1][ws];
  }
  if (h->nbr[1]) {
    x.hi = h->ghost[1][rs];
    x.put_hi = h->nbr[1]->ghost[0][ws];
  }
  // distributed: neighbours' ghosts + arrival counters (device-side sync)
  for (int s = 0; s < 2; ++s) {
    if (!h->peer[s].linked) continue;
    if (s == 0) {
      x.lo = h->ghost[0][rs];
      x.put_lo = h->peer[0].ghost[ws];
      x.sig_lo = h->peer[0].cnt;
      x.wait_lo = h->cnt;
      x.expect_lo = h->recv[0];
    } else {
      x.hi = h->ghost[1][rs];
      x.put_hi = h->peer[1].ghost[ws];
      x.sig_hi = h->peer[1].cnt;
      x.wait_hi = h->cnt + 1;
      x.expect_hi = h->recv[1];
    }
    x.timeout_flag = h->d_event;
  }
  return x;
}

bool dist_linked(const emrkc_handle* h) { return h->peer[0].linked || h->peer[1].linked; }

// After a level: the neighbours ran the same kernel family on the same x-y
// geometry, so each sends the same number of arrivals.
void dist_account(emrkc_handle* h, long long signals) {
  for (int s = 0; s < 2; ++s)
    if (h->peer[s].linked) h->recv[s] += static_cast<unsigned long long>(signals);
}

// One step of the plan, launched level by level (a level = one stencil
// consuming kernel). No host synchronisation.
struct StepCtx {
  int in = 0;
  int w[3] = {0, 0, 0};
  int nw = 1;
  double t = 0.0;
  StageArgs a{};
};

void begin_step(emrkc_handle* h, double t, long long step_in_run,
                unsigned long long* gate_slot, StepCtx* c) {
  const Plan& pl = h->plan;
  c->in = h->cur;
  c->t = t;
  c->nw = (pl.s == 1) ? 1 : (pl.s == 2 ? 2 : 3);
  for (int k = 0; k < c->nw; ++k) c->w[k] = (c->in + 1 + k) % h->nbuf;
  const unsigned long long stride =
      static_cast<unsigned long long>(pl.s) * (pl.m + 1) + 2;
  StageArgs& a = c->a;
  a = StageArgs{};
  a.eta = pl.eta;
  a.inv_eta = 1.0 / pl.eta;
  a.s = pl.s;
  a.m = pl.m;
  a.in_mueta = h->d_coef;
  a.in_nu = h->d_coef + (pl.m + 1);
  a.in_kappa = h->d_coef + 2 * (pl.m + 1);
  a.code_base = static_cast<unsigned long long>(step_in_run) * stride;
  a.event = h->d_event;
  a.gate_slot = gate_slot;
  // run loops keep consecutive per-step slots and the initial state's slot
  // (slot_init); single steps have no earlier range
  a.gate_prev = !h->slot_init ? nullptr : (step_in_run > 0 ? gate_slot - 2 : h->slot_init);
  a.fs = h->fs;
  a.ye = h->ye;
  for (int k = 0; k < 3; ++k) a.u[k] = h->u[k];
}

// ---- TMA descriptors -------------------------------------------------------
// Tensor maps over the SoA state (P/include/mrkc/monodomain.hpp:51-60 layout):
// spatial dims (n0, n1, nzl) [2-D: (n0, nzl)], plus the field axis of stride
// nn for the gate boxes. Encoded through the driver entry point (no -lcuda).
enum TmaKind { kTmaHalo = 0, kTmaCenter = 1, kTmaGates = 2, kTmaAll = 3, kTmaGhost = 4 };

PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// TMA needs 16-byte global strides (n0 even) and a 2-D or 3-D grid.
bool tma_supported(const emrkc_handle* h) {
  return h->geom.dim >= 2 && h->geom.n0 % 2 == 0 && tma_encoder() != nullptr;
}

// rmul: tile rows x rmul (the multi-row inner-stage kernel, vin_rows);
// xmul: tile width x xmul (3-D; the pair-per-thread node kernel)
int tma_map(emrkc_handle* h, const void* ptr, int kind, CUtensorMap* out, int rmul = 1,
            int xmul = 1) {
  const int key = kind + 1000 * (rmul - 1) + 100000 * (xmul - 1);
  for (const auto& e : h->tmaps)
    if (e.ptr == ptr && e.kind == key) {
      *out = e.map;
      return EMRKC_OK;
    }
  const Geom& g = h->geom;
  const bool d3 = g.dim == 3;
  const cuuint32_t tx = d3 ? emrkc_k::kTX3 * static_cast<cuuint32_t>(xmul) : emrkc_k::kTX2,
                   ty = d3 ? emrkc_k::kTY3 * static_cast<cuuint32_t>(rmul) : 1;
  const bool halo = kind == kTmaHalo || kind == kTmaGhost;
  cuuint64_t dims[4];
  cuuint64_t strides[3];
  cuuint32_t box[4], es[4] = {1, 1, 1, 1};
  cuuint32_t rank = 0;
  dims[rank] = static_cast<cuuint64_t>(g.n0);
  box[rank++] = halo ? tx + 4 : tx;  // x0-2 .. x0+tx+1: 16-byte aligned start
  if (d3) {
    strides[rank - 1] = sizeof(double) * static_cast<cuuint64_t>(g.n0);
    dims[rank] = static_cast<cuuint64_t>(g.n1);
    box[rank++] = halo ? ty + 2 : ty;
  }
  if (kind != kTmaGhost) {
    strides[rank - 1] = sizeof(double) * static_cast<cuuint64_t>(g.plane);
    dims[rank] = static_cast<cuuint64_t>(g.nzl);
    box[rank++] = 1;
  }
  if (kind == kTmaGates || kind == kTmaAll) {  // gates (+ aux) from field 1 / all fields
    strides[rank - 1] = sizeof(double) * static_cast<cuuint64_t>(g.nn);
    dims[rank] = static_cast<cuuint64_t>(g.nf);
    box[rank++] = static_cast<cuuint32_t>(kind == kTmaGates ? g.nf - 1 : g.nf);
  }
  if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0)
    return set_err(h, EMRKC_ECUDA, "TMA: buffer %p not 16-byte aligned", ptr);
  CUtensorMap m;
  const CUresult r = tma_encoder()(
      &m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(ptr), dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(h, EMRKC_ECUDA, "cuTensorMapEncodeTiled failed (%d, kind %d)", (int)r, kind);
  h->tmaps.push_back({ptr, key, m});
  *out = m;
  return EMRKC_OK;
}

// 3-D map over one V-sized field (n0, n1, nzl) with box (bx, by, 1); key
// distinguishes box shapes in the cache (>= 100).
// k_fused2 boxes: kind 0 = V with halo (kFuTX + 4, kFuTY + 2, 1), kind 1 =
// the three gate fields (kFuTX, kFuTY, 1, 3) from field 1.
int tma_map_fused(emrkc_handle* h, const void* ptr, int kind, CUtensorMap* out) {
  const int key = 3000 + kind;
  for (const auto& e : h->tmaps)
    if (e.ptr == ptr && e.kind == key) {
      *out = e.map;
      return EMRKC_OK;
    }
  const Geom& g = h->geom;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(g.n0), static_cast<cuuint64_t>(g.n1),
                              static_cast<cuuint64_t>(g.nzl), 4};
  const cuuint64_t strides[3] = {sizeof(double) * static_cast<cuuint64_t>(g.n0),
                                 sizeof(double) * static_cast<cuuint64_t>(g.plane),
                                 sizeof(double) * static_cast<cuuint64_t>(g.nn)};
  const cuuint32_t box[4] = {
      static_cast<cuuint32_t>(kind == 0 ? emrkc_k::kFuTX + 4 : emrkc_k::kFuTX),
      static_cast<cuuint32_t>(kind == 0 ? emrkc_k::kFuTY + 2 : emrkc_k::kFuTY), 1, 3};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0)
    return set_err(h, EMRKC_ECUDA, "TMA: buffer %p not 16-byte aligned", ptr);
  CUtensorMap m;
  const CUresult r = tma_encoder()(
      &m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, kind == 0 ? 3 : 4, const_cast<void*>(ptr), dims,
      strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(h, EMRKC_ECUDA, "cuTensorMapEncodeTiled failed (%d, fused %d)", (int)r, kind);
  h->tmaps.push_back({ptr, key, m});
  *out = m;
  return EMRKC_OK;
}

int tma_map_box3(emrkc_handle* h, const void* ptr, cuuint32_t bx, cuuint32_t by, int key,
                 CUtensorMap* out, int64_t nz = -1) {
  for (const auto& e : h->tmaps)
    if (e.ptr == ptr && e.kind == key) {
      *out = e.map;
      return EMRKC_OK;
    }
  const Geom& g = h->geom;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.n0), static_cast<cuuint64_t>(g.n1),
                              static_cast<cuuint64_t>(nz >= 0 ? nz : g.nzl)};
  const cuuint64_t strides[2] = {sizeof(double) * static_cast<cuuint64_t>(g.n0),
                                 sizeof(double) * static_cast<cuuint64_t>(g.plane)};
  const cuuint32_t box[3] = {bx, by, 1}, es[3] = {1, 1, 1};
  if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0)
    return set_err(h, EMRKC_ECUDA, "TMA: buffer %p not 16-byte aligned", ptr);
  CUtensorMap m;
  const CUresult r = tma_encoder()(
      &m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(ptr), dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(h, EMRKC_ECUDA, "cuTensorMapEncodeTiled failed (%d, key %d)", (int)r, key);
  h->tmaps.push_back({ptr, key, m});
  *out = m;
  return EMRKC_OK;
}

// Pair-per-thread node kernel (k_node_pair): 3-D handles (whole grid or
// slab) on the TMA path with HH proper (no aux rows); EMRKC_PAIR=0 keeps
// k_node_tma.
bool use_pair(const emrkc_handle* h) {
  return h->pair && h->fast && h->pipe == 3 && h->geom.dim == 3 && h->geom.naux == 0;
}

// Temporally blocked inner stages (k_vin_tb) apply: 3-D handle on the TMA
// path with 2 <= K = m - 1 <= kTbMaxK (default; EMRKC_TB=0 disables). Slabs exchange
// K planes of d_1 (the wide halo), so every slab of the partition must be at
// least K planes deep (min_depth: emrkc_set_slab_min_depth, or the group).
bool use_tb(const emrkc_handle* h, const Plan& pl) {
  const int K = pl.m - 1;
  // K = 1 (m = 2: the single inner stage through k_vin_tb's lean march instead of
  // k_vin_tma_r) only with EMRKC_TB=2 (A/B)
  if (!(h->tb && h->pipe == 3 && h->geom.dim == 3 && K >= (h->tb >= 2 ? 1 : 2) &&
        K <= emrkc_k::kTbMaxK))
    return false;
  return !h->partitioned || h->min_depth >= K;
}

// Fused s = 1, m = 2 step (k_fused2): whole-grid 3-D handles on the TMA
// path whose plane splits into >= 90% of the co-resident block slots
// (ntx = n0 / 64 column tiles of width 64, nty tile rows of <= 14 rows,
// nzc z-chunks of >= 8 planes).
bool fused_plan(emrkc_handle* h) {
  if (h->fu_planned) return h->fu_ntx > 0;
  h->fu_planned = true;
  const Geom& g = h->geom;
  if (g.dim != 3 || g.n0 % emrkc_k::kFuTX || g.n1 < 2 * emrkc_k::kFuTY || g.nzl < 8) return false;
  const int per_sm = emrkc_k::fused_blocks_per_sm();
  int sms = 0;
  if (per_sm < 1 || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device) !=
                        cudaSuccess)
    return false;
  const int slots = per_sm * sms;
  const int ntx = g.n0 / emrkc_k::kFuTX;
  const int ny_min = (g.n1 + emrkc_k::kFuTY - 1) / emrkc_k::kFuTY;
  int best = 0, bty = 0, bz = 0;
  for (int nzc = 1; nzc <= 16 && g.nzl / nzc >= 8; ++nzc)
    for (int nty = ny_min; nty <= g.n1 / 2; ++nty) {
      const long long tiles = (long long)ntx * nty * nzc;
      if (tiles > slots) break;
      if (tiles > best) {
        best = static_cast<int>(tiles);
        bty = nty;
        bz = nzc;
      }
    }
  if (best < 0.9 * slots) return false;
  const size_t xn = static_cast<size_t>(best) * 4 * 4 * emrkc_k::kFuTX;
  if (cudaMalloc(&h->fu_xch, sizeof(double) * xn) != cudaSuccess ||
      cudaMalloc(&h->fu_flags, sizeof(unsigned long long) * best) != cudaSuccess ||
      cudaMemset(h->fu_flags, 0, sizeof(unsigned long long) * best) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  h->fu_ntx = ntx;
  h->fu_nty = bty;
  h->fu_nzc = bz;
  return true;
}

bool use_fused(emrkc_handle* h, const Plan& pl) {
  return h->fused && h->fast && h->pipe == 3 && !h->partitioned && h->zr_lo < 0 &&
         h->geom.naux == 0 &&
         h->geom.dim == 3 && pl.s == 1 && pl.m == 2 && !pl.exex && pl.method != kMethodMrkc &&
         fused_plan(h);
}

// The neighbours' d_1 ghosts this handle's inner-stage-1 kernel stores into
// (side 0: the lower neighbour's upper ghost), parity par.
double* nbr_dghost(const emrkc_handle* h, int side, int par) {
  if (h->nbr[side]) return h->nbr[side]->dghost[1 - side][par];
  if (h->peer[side].linked) return h->peer[side].dghost[par];
  return nullptr;
}

int tma_ghosts(emrkc_handle* h, const Halo& hl, CUtensorMap* lo, CUtensorMap* hi, int rmul = 1,
               int xmul = 1) {
  std::memset(lo, 0, sizeof *lo);
  std::memset(hi, 0, sizeof *hi);
  if (hl.lo) {
    const int rc = tma_map(h, hl.lo, kTmaGhost, lo, rmul, xmul);
    if (rc) return rc;
  }
  if (hl.hi) {
    const int rc = tma_map(h, hl.hi, kTmaGhost, hi, rmul, xmul);
    if (rc) return rc;
  }
  return EMRKC_OK;
}

// FastArgs of the node level (inner stage 1) of outer stage j: pointers and
// coefficients from the step context.
void fill_node_args(emrkc_handle* h, const Plan& pl, const StageArgs& a, int j,
                    emrkc_k::FastArgs* f) {
  const double cG = pl.mudt[j] / pl.eta;
  f->g1 = a.g1;
  f->g2 = a.g2;
  f->out = a.out;
  f->fs = h->fs;
  f->u1 = h->u[3];
  f->eta = pl.eta;
  f->stim = a.stim;
  f->cG = cG * pl.gate_c;  // gate rows (progressive: c_m (y_E - z))
  f->cV = cG * pl.in_mueta[1];
  f->mue1 = pl.in_mueta[1];
  f->exex = pl.exex;
  f->z_lo = h->zr_lo >= 0 ? h->zr_lo : 0;  // plane range (pipelined host step)
  f->z_hi = h->zr_lo >= 0 ? h->zr_hi : h->geom.nzl;
  f->nu = a.nu;
  f->kappa = a.kappa;
  // aux rows (EMRKC_MODEL_HH_AUX): the inner iterate is z + c_m eta g_S
  f->cA = pl.mudt[j] * pl.inner.c[pl.m];
  // fast ionic path only where its range analysis holds (fast_math.cuh)
  fast_window(pl.eta, &f->vmid, &f->vfast);
  {
    const double vlo = f->vmid - f->vfast, vhi = f->vmid + f->vfast;
    auto hiword = [](double x) {
      uint64_t b = 0;
      std::memcpy(&b, &x, sizeof b);
      return static_cast<uint32_t>(b >> 32);
    };
    f->vq_pos = 0;
    f->vq_neg = 0;
    if (vlo < 0.0 && vhi > 0.0 && std::isfinite(vlo) && std::isfinite(vhi)) {
      f->vq_pos = static_cast<int>(hiword(vhi));
      f->vq_neg = 0x80000000u + hiword(-vlo);
    }
  }
  f->j = j;
  f->m = pl.m;
  f->s = pl.s;
  f->last = a.last;
  f->zc = h->zc;
  f->code_base = a.code_base;
  f->event = a.event;
  f->gate_slot = a.gate_slot;
  f->gate_prev = a.last ? a.gate_prev : nullptr;
}

// Launches inner stage k (1..m) of outer stage j (1..s).
int launch_level(emrkc_handle* h, StepCtx* c, int j, int k) {
  const Plan& pl = h->plan;
  StageArgs& a = c->a;
  const int nw = c->nw;
  a.j = j;
  a.last = (j == pl.s);
  a.out = h->buf[c->w[(j - 1) % nw]];
  a.g1 = (j == 1) ? h->buf[c->in] : h->buf[c->w[(j - 2) % nw]];
  a.g2 = (j == 1) ? nullptr
                  : (j == 2 ? h->buf[c->in] : h->buf[c->w[(j - 3) % nw]]);
  a.mudt = pl.mudt[j];
  a.nu = pl.outer.nu[j];
  a.kappa = pl.outer.kappa[j];
  // stage time: t for j = 1, t + c_{j-1} dt after (P/src/cheb.cpp:90,97)
  const double r = (j == 1) ? c->t : c->t + pl.outer.c[j - 1] * pl.dt;
  a.stim = stim_rate_at(&h->p, r);
  const Halo hl = halo_at(h, h->level);
  if (pl.method == kMethodMrkc) {
    emrkc_k::MrkcArgs f{};
    f.g1 = a.g1;
    f.g2 = a.g2;
    f.out = a.out;
    f.fs = h->mr_fs;
    f.um1 = k == 1 ? a.g1 : h->mr_u[(k - 1) % 3];
    f.um2 = k == 2 ? a.g1 : (k > 2 ? h->mr_u[(k - 2) % 3] : nullptr);
    f.uk = h->mr_u[k % 3];
    f.eta = pl.eta;
    f.mueta = pl.in_mueta[k];
    f.nu = pl.inner.nu[k];
    f.kappa = pl.inner.kappa[k];
    f.mudt = pl.mudt[j];
    f.onu = a.nu;
    f.okappa = a.kappa;
    f.stim = a.stim;
    f.stiff = h->stiff;
    f.j = j;
    f.k = k;
    f.m = pl.m;
    f.s = pl.s;
    f.last = a.last;
    f.code_base = a.code_base;
    f.event = a.event;
    CK(h, emrkc_k::launch_mrkc_stage(h->geom, f, lstream(h)));
    if (a.last && k == pl.m)  // gate range of the step's result (simulate.cpp:228)
      CK(h, emrkc_k::launch_gate_range(h->geom, a.out, a.gate_slot, lstream(h)));
    ++h->level;
    return EMRKC_OK;
  }
  if (h->fast) {
    const double cG = pl.mudt[j] / pl.eta;
    // arrivals this level sends each neighbour (cross-process protocol)
    long long signals = h->pipe && h->geom.dim >= 2 ? emrkc_k::halo_signals_pipe(h->geom)
                                                     : emrkc_k::halo_signals_march(h->geom);
    if (use_tb(h, pl) && k > 2) return EMRKC_OK;  // fused into level k == 2: no level
    if (k == 2 && use_fused(h, pl)) return EMRKC_OK;  // ran inside the k == 1 launch
    if (k == 1) {
      emrkc_k::FastArgs f{};
      fill_node_args(h, pl, a, j, &f);
      if (use_fused(h, pl)) {
        // the whole step (levels 1 and 2) in one persistent pass
        emrkc_k::FusedArgs fa{};
        fa.f = f;
        fa.inv_mue1 = 1.0 / pl.in_mueta[1];
        fa.mueta2 = pl.in_mueta[2];
        fa.nu2 = pl.inner.nu[2];
        fa.cG2 = cG;
        fa.xch = h->fu_xch;
        fa.flags = h->fu_flags;
        h->fu_epoch += 1ull << 32;
        fa.epoch = h->fu_epoch;
        fa.ntx = h->fu_ntx;
        fa.nty = h->fu_nty;
        fa.nzc = h->fu_nzc;
        emrkc_k::TmaFused tm;
        int rc = tma_map_fused(h, f.g1, 0, &tm.v);
        if (!rc) rc = tma_map_fused(h, f.g1, 1, &tm.gates);
        if (rc) return rc;
        CK(h, emrkc_k::launch_fused2(h->geom, fa, tm, lstream(h)));
        ++h->level;
        return EMRKC_OK;
      }
      const int pzc = use_pair(h) ? emrkc_k::pair_zc(h->geom, j == 1, h->pair == 2) : 0;
      Halo hn = hl;
      if (h->pipe == 3 && h->partitioned && use_tb(h, pl)) {
        // wide halo: K planes of d_1 into the neighbours' d_1 ghosts
        const int par = static_cast<int>(h->kstage & 1);
        hn.put_lo = hn.put_hi = nullptr;
        hn.kput = pl.m - 1;
        hn.kput_lo = hl.put_lo ? nbr_dghost(h, 0, par) : nullptr;
        hn.kput_hi = hl.put_hi ? nbr_dghost(h, 1, par) : nullptr;
        signals = emrkc_k::halo_signals_pipe(h->geom) * hn.kput;
      }
      if (pzc > 0) {
        // pair-per-thread node kernel (3-D, HH proper)
        emrkc_k::TmaNode tm;
        std::memset(&tm, 0, sizeof tm);
        const int xm = emrkc_k::pair_tx(h->geom) / emrkc_k::kTX3, rm = 2 / xm;  // 64 x 4 or 32 x 8
        int rc = tma_map(h, f.g1, kTmaHalo, &tm.v, rm, xm);
        if (!rc) rc = tma_map(h, f.g1, kTmaGates, &tm.gates, rm, xm);
        if (!rc && f.g2) rc = tma_map(h, f.g2, kTmaAll, &tm.g2, rm, xm);
        if (!rc) rc = tma_ghosts(h, hl, &tm.glo, &tm.ghi, rm, xm);
        if (rc) return rc;
        f.zc = pzc;
        CK(h, emrkc_k::launch_node_pair(h->geom, hn, f, tm, pl.m >= 2, lstream(h)));
      } else if (h->pipe == 3) {
        emrkc_k::TmaNode tm;
        int rc = tma_map(h, f.g1, kTmaHalo, &tm.v);
        if (!rc) rc = tma_map(h, f.g1, kTmaGates, &tm.gates);
        if (!rc && f.g2) rc = tma_map(h, f.g2, kTmaAll, &tm.g2);
        if (!f.g2) std::memset(&tm.g2, 0, sizeof tm.g2);
        if (!rc) rc = tma_ghosts(h, hl, &tm.glo, &tm.ghi);
        if (rc) return rc;
        CK(h, emrkc_k::launch_node_tma(h->geom, hn, f, tm, pl.m >= 2, lstream(h)));
      } else if (h->pipe == 2)
        CK(h, emrkc_k::launch_node_persist(h->geom, hl, f, pl.m >= 2, lstream(h)));
      else if (h->pipe)
        CK(h, emrkc_k::launch_node_pipe(h->geom, hl, f, pl.m >= 2, lstream(h)));
      else
        CK(h, emrkc_k::launch_node_fast(h->geom, hl, f, pl.m >= 2, lstream(h)));
    } else if (use_tb(h, pl)) {
      // stages 2..m in one pass at k == 2; levels k > 2 launch nothing
      if (k == 2) {
        emrkc_k::TbArgs f{};
        for (int kk = 0; kk <= pl.m; ++kk) {
          f.mueta[kk] = pl.in_mueta[kk];
          f.nu[kk] = pl.inner.nu[kk];
          f.kappa[kk] = pl.inner.kappa[kk];
        }
        f.g1v = a.g1;
        f.g2v = a.g2;
        f.outv = a.out;
        f.inv_mue1 = 1.0 / pl.in_mueta[1];
        f.onu = a.nu;
        f.okappa = a.kappa;
        f.cG = cG;
        f.j = j;
        f.m = pl.m;
        f.s = pl.s;
        f.last = a.last;
        const int K = pl.m - 1;
        f.zc = emrkc_k::tb_zc(h->geom, K);
        f.code_base = a.code_base;
        f.event = a.event;
        emrkc_k::TmaTb tm;
        std::memset(&tm, 0, sizeof tm);
        const cuuint32_t bx = emrkc_k::kTbTX + 2 * emrkc_k::tb_hx(K), by = emrkc_k::kTbTY + 2 * K;
        int rc = tma_map_box3(h, h->u[3], bx, by, 100 + K, &tm.d1);
        // slabs: this handle's d_1 ghosts (K planes per face with a neighbour)
        Halo ht = hl;
        ht.lo = ht.hi = nullptr;
        const int par = static_cast<int>(h->kstage & 1);
        if (hl.lo) {
          ht.lo = h->dghost[0][par];
          if (!rc) rc = tma_map_box3(h, ht.lo, bx, by, 200 + K, &tm.d1lo, K);
        }
        if (hl.hi) {
          ht.hi = h->dghost[1][par];
          if (!rc) rc = tma_map_box3(h, ht.hi, bx, by, 200 + K, &tm.d1hi, K);
        }
        if (rc) return rc;
        CK(h, emrkc_k::launch_vin_tb(h->geom, ht, f, tm, lstream(h)));
        ++h->kstage;
        signals = emrkc_k::halo_signals_tb(h->geom);
      }
    } else {
      emrkc_k::FastInnerArgs f{};
      // increment form: d_1 stays in u[3] (it also gives a = d_1/(mu'_1 eta)),
      // d_k (k >= 2) rotates through u[0..2]
      auto dbuf = [&](int kk) { return kk == 1 ? h->u[3] : h->u[(kk - 2) % 3]; };
      f.um1 = dbuf(k - 1);
      f.um2 = (k == 2) ? nullptr : dbuf(k - 2);
      f.d1 = h->u[3];
      f.inv_mue1 = 1.0 / pl.in_mueta[1];
      f.uk = dbuf(k);
      f.g1v = a.g1;
      f.g2v = a.g2;
      f.outv = a.out;
      f.mueta = pl.in_mueta[k];
      f.nu = pl.inner.nu[k];
      f.kappa = pl.inner.kappa[k];
      f.onu = a.nu;
      f.okappa = a.kappa;
      f.cG = cG;
      f.j = j;
      f.k = k;
      f.m = pl.m;
      f.s = pl.s;
      f.last = a.last;
      f.zc = h->zc;
      f.z_lo = h->zr_lo >= 0 ? h->zr_lo : 0;  // plane range (pipelined host step)
      f.z_hi = h->zr_lo >= 0 ? h->zr_hi : h->geom.nzl;
      f.code_base = a.code_base;
      f.event = a.event;
      if (h->pipe == 3) {
        emrkc_k::TmaVin tm;
        std::memset(&tm, 0, sizeof tm);
        const int rm = emrkc_k::vin_rows(h->geom);
        int rc = tma_map(h, f.um1, kTmaHalo, &tm.u, rm);
        if (!rc) rc = tma_map(h, f.d1, kTmaCenter, &tm.d1, rm);
        if (!rc && f.um2) rc = tma_map(h, f.um2, kTmaCenter, &tm.um2, rm);
        if (!rc && k == pl.m) rc = tma_map(h, f.g1v, kTmaCenter, &tm.g1v, rm);
        if (!rc && k == pl.m && f.g2v) rc = tma_map(h, f.g2v, kTmaCenter, &tm.g2v, rm);
        if (!rc) rc = tma_ghosts(h, hl, &tm.glo, &tm.ghi, rm);
        if (rc) return rc;
        CK(h, emrkc_k::launch_vin_tma(h->geom, hl, f, tm, lstream(h)));
        signals = emrkc_k::halo_signals_vin(h->geom);
      } else if (h->pipe)
        CK(h, emrkc_k::launch_vin_pipe(h->geom, hl, f, lstream(h)));
      else
        CK(h, emrkc_k::launch_vin_fast(h->geom, hl, f, lstream(h)));
    }
    if (dist_linked(h)) dist_account(h, signals);
  } else if (pl.m == 1) {
    CK(h, emrkc_k::launch_stage_m1(h->geom, hl, a, 0, lstream(h)));
  } else if (k == 1) {
    CK(h, emrkc_k::launch_stage_first(h->geom, hl, a, 0, lstream(h)));
  } else {
    CK(h, emrkc_k::launch_stage_inner(h->geom, hl, a, k, 0, lstream(h)));
  }
  ++h->level;
  return EMRKC_OK;
}

int end_step(emrkc_handle* h, const StepCtx* c) {
  return c->w[(h->plan.s - 1) % c->nw];
}

// z-pipelined step (s = 1, m >= 2, whole grid, TMA kernels): the node kernel
// (level 1) runs in EMRKC_ZPIPE z-chunks on the handle's stream, and level
// k >= 2 of chunk c runs on a second stream as soon as level k - 1 of chunk
// c is done, its plane range lagging by k planes (plane p of level k needs
// level k - 1 at p + 1; the ranges of emrkc_step_host). The node kernel is
// FP64-issue bound and the inner stages HBM bound, so the two overlap on the
// SMs; the results are the unpipelined step's bit for bit.
bool use_zpipe(emrkc_handle* h, const Plan& pl) {
  const int K = h->zpipe;
  return K > 1 && !h->partitioned && h->fast && h->pipe == 3 && pl.s == 1 && pl.m >= 2 &&
         pl.method != kMethodMrkc && !pl.exex && !use_tb(h, pl) && !use_fused(h, pl) &&
         h->zr_lo < 0 && !h->level_hook && h->geom.nzl >= (pl.m + 1) * K;
}

int enqueue_step_zpipe(emrkc_handle* h, double t, long long step_in_run,
                       unsigned long long* gate_slot, int* out_idx) {
  const int K = h->zpipe;
  if (!h->s_aux) {
    CK(h, cudaStreamCreateWithFlags(&h->s_aux, cudaStreamNonBlocking));
    h->zp_ev.resize(64);
    for (auto& e : h->zp_ev) CK(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(h, cudaEventCreateWithFlags(&h->zp_join, cudaEventDisableTiming));
  }
  const Plan& pl = h->plan;
  const int nz = h->geom.nzl, m = pl.m;
  auto zc = [&](int c) { return static_cast<int>(static_cast<int64_t>(c) * nz / K); };
  auto kr = [&](int c, int k) { return c == 0 ? 0 : (c == K ? nz : zc(c) - k); };
  StepCtx c;
  begin_step(h, t, step_in_run, gate_slot, &c);
  // the second stream starts behind everything enqueued so far
  CK(h, cudaEventRecord(h->zp_join, h->stream));
  CK(h, cudaStreamWaitEvent(h->s_aux, h->zp_join, 0));
  int rc = EMRKC_OK;
  for (int q = 0; q <= K && !rc; ++q) {
    if (q < K) {  // node kernel, chunk q
      h->ls = h->stream;
      h->zr_lo = kr(q, 1);
      h->zr_hi = kr(q + 1, 1);
      rc = launch_level(h, &c, 1, 1);
      if (!rc) CK(h, cudaEventRecord(h->zp_ev[q], h->stream));
    }
    if (q >= 1 && !rc) {  // inner stages, chunk q - 1
      CK(h, cudaStreamWaitEvent(h->s_aux, h->zp_ev[q - 1], 0));
      h->ls = h->s_aux;
      for (int k = 2; k <= m && !rc; ++k) {
        h->zr_lo = kr(q - 1, k);
        h->zr_hi = kr(q, k);
        rc = launch_level(h, &c, 1, k);
      }
    }
  }
  h->ls = nullptr;
  h->zr_lo = h->zr_hi = -1;
  // the handle's stream continues behind the whole step
  CK(h, cudaEventRecord(h->zp_join, h->s_aux));
  CK(h, cudaStreamWaitEvent(h->stream, h->zp_join, 0));
  if (rc) return rc;
  *out_idx = end_step(h, &c);
  return EMRKC_OK;
}

// Cross-step fusion (k_step_x, EMRKC_XSTEP=1): in a run loop of a 3-D whole
// grid with s = 1, m = 2 (emRKC standard), inner stage 2 of step r and the
// node update of step r + 1 run as one launch. The state needs three
// buffers (y_r stays intact for the abort rollback while y_{r+1} and the
// gates of y_{r+2} are written) and d_1 two (u[3] / u[0], swapped per launch).
bool use_xstep(emrkc_handle* h, const Plan& pl, int64_t nsteps) {
  return h->xstep && use_pair(h) && !h->partitioned && !h->level_hook && h->zr_lo < 0 &&
         pl.s == 1 && pl.m == 2 && pl.method != kMethodMrkc && !pl.exex && pl.gate_c == 1.0 &&
         nsteps >= 2 && !use_fused(h, pl) && !use_zpipe(h, pl) && emrkc_k::pair_tx(h->geom) == 64 &&
         emrkc_k::pair_zc(h->geom, true, h->pair == 2) > 0;
}

// c: step r (its node level is done, its inner stage 2 runs here); cn: step
// r + 1 after begin_step (cn->in == c->w[0]).
int launch_xstep(emrkc_handle* h, const StepCtx* c, StepCtx* cn) {
  const Plan& pl = h->plan;
  StageArgs& a = cn->a;
  a.j = 1;
  a.last = 1;
  a.out = h->buf[cn->w[0]];
  a.g1 = h->buf[cn->in];
  a.g2 = nullptr;
  a.mudt = pl.mudt[1];
  a.nu = pl.outer.nu[1];
  a.kappa = pl.outer.kappa[1];
  a.stim = stim_rate_at(&h->p, cn->t);
  emrkc_k::XArgs x{};
  fill_node_args(h, pl, a, 1, &x.f);
  x.f.u1 = h->u[0];  // d_1 of step r + 1 (u[3] holds step r's until the swap below)
  x.f.zc = emrkc_k::pair_zc(h->geom, true, h->pair == 2);
  x.vn = h->buf[c->in];
  x.d1 = h->u[3];
  x.vout = h->buf[c->w[0]];
  x.inv_mue1 = 1.0 / pl.in_mueta[1];
  x.mueta2 = pl.in_mueta[2];
  x.nu2 = pl.inner.nu[2];
  x.cG2 = pl.mudt[1] / pl.eta;
  x.code_prev = c->a.code_base;
  emrkc_k::TmaX tm;
  std::memset(&tm, 0, sizeof tm);
  int rc = tma_map_box3(h, h->u[3], emrkc_k::kTX3 * emrkc_k::kPairXMul + 4, emrkc_k::kTY3 + 4, 150,
                        &tm.d1);
  if (!rc) rc = tma_map(h, a.g1, kTmaGates, &tm.gates, 1, emrkc_k::kPairXMul);
  if (rc) return rc;
  CK(h, emrkc_k::launch_step_x(h->geom, x, tm, lstream(h)));
  std::swap(h->u[3], h->u[0]);
  h->level += 2;
  return EMRKC_OK;
}

int enqueue_step(emrkc_handle* h, double t, long long step_in_run,
                 unsigned long long* gate_slot, int* out_idx) {
  if (use_zpipe(h, h->plan)) return enqueue_step_zpipe(h, t, step_in_run, gate_slot, out_idx);
  StepCtx c;
  begin_step(h, t, step_in_run, gate_slot, &c);
  for (int j = 1; j <= h->plan.s; ++j)
    for (int k = 1; k <= h->plan.m; ++k) {
      const int rc = launch_level(h, &c, j, k);
      if (rc) return rc;
      if (h->level_hook) {  // lockstep across processes (testing aid)
        CK(h, cudaStreamSynchronize(h->stream));
        h->level_hook(h->level_ctx);
      }
    }
  *out_idx = end_step(h, &c);
  return EMRKC_OK;
}

struct Decoded {
  bool none = true;
  bool guard = false;
  long long step = -1;
  int outer_stage = 0, stage = 0, inner = 0;
};

Decoded decode_event(unsigned long long ev, const Plan& pl) {
  Decoded d;
  if (ev == kNoEvent || ev == 0) return d;  // 0: protocol timeout (checked by callers)
  const unsigned long long stride =
      static_cast<unsigned long long>(pl.s) * (pl.m + 1) + 2;
  d.none = false;
  d.step = static_cast<long long>(ev / stride);
  const int ord = static_cast<int>(ev % stride);
  if (ord == pl.s * (pl.m + 1) + 1) {
    d.guard = true;
    return d;
  }
  d.outer_stage = (ord - 1) / (pl.m + 1) + 1;
  const int k = (ord - 1) % (pl.m + 1) + 1;
  if (k <= pl.m) {
    d.inner = 1;
    d.stage = k;
  } else {
    d.inner = 0;
    d.stage = d.outer_stage;
  }
  return d;
}

// Work tallies of a step aborted at (outer stage j, inner stage k):
// the reference counts calls made before the throw (P/src/multirate.cpp:18-38).
void partial_counters(const Decoded& d, const Plan& pl, int64_t* fF,
                      int64_t* fS, int64_t* ex) {
  const int j = d.outer_stage;
  *ex += exp_per_step(pl.method, j);
  *fS += j;
  *fF += static_cast<int64_t>(j - 1) * pl.m + (d.inner ? d.stage : pl.m);
}

int init_handle(emrkc_handle* h) {
  CK(h, cudaSetDevice(h->device));
  CK(h, cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  CK(h, cudaMalloc(&h->d_event, sizeof(unsigned long long)));
  CK(h, cudaMalloc(&h->d_red, sizeof(double) * (emrkc_k::power_blocks() + 8)));
  CK(h, cudaEventCreate(&h->ev0));
  CK(h, cudaEventCreate(&h->ev1));
  if (h->partitioned) {
    const size_t pl = static_cast<size_t>(h->geom.plane);
    const size_t np = arena_planes(h->geom.dim);
    h->arena_bytes = sizeof(double) * np * pl + 256;
    CK(h, cudaMalloc(&h->arena, h->arena_bytes));
    CK(h, cudaMemset(h->arena, 0, h->arena_bytes));
    double* base = static_cast<double*>(h->arena);
    for (int s = 0; s < 2; ++s)
      for (int k = 0; k < 2; ++k) {
        h->ghost[s][k] = base + (2 * s + k) * pl;
        if (h->geom.dim == 3) h->dghost[s][k] = dghost_at(base, pl, s, k);
      }
    h->cnt = reinterpret_cast<unsigned long long*>(base + np * pl);
  }
  const char* f = std::getenv("EMRKC_FAST");
  h->fast = f ? std::atoi(f) : 1;
  h->zc = emrkc_k::fast_zc(h->geom);
  const char* pp = std::getenv("EMRKC_PIPE");
  // 3: TMA-staged blocks, 1: cp.async-staged blocks, 2: persistent cp.async
  // node kernel, 0: march
  h->pipe = (pp && *pp) ? std::atoi(pp) : 3;
  if (h->pipe == 3 && !tma_supported(h)) h->pipe = 1;
  if (h->pipe != 3) h->zc = std::min(h->zc, emrkc_k::kMaxZcPipe);
  if (const char* tb = std::getenv("EMRKC_TB"))
    if (*tb) h->tb = std::max(0, std::min(2, std::atoi(tb)));
  if (const char* xs = std::getenv("EMRKC_XSTEP"))
    if (*xs) h->xstep = std::atoi(xs) != 0;
  if (const char* pr = std::getenv("EMRKC_PAIR"))
    if (*pr) h->pair = std::max(0, std::min(2, std::atoi(pr)));  // 2: also on small grids (tests)
  if (const char* fu = std::getenv("EMRKC_FUSED"))
    if (*fu) h->fused = std::atoi(fu) != 0;
  if (const char* zp = std::getenv("EMRKC_ZPIPE"))
    if (*zp) h->zpipe = std::max(0, std::min(64, std::atoi(zp)));
  if (const char* zc = std::getenv("EMRKC_ZC"))
    if (*zc)
      h->zc = std::min(h->pipe == 3 ? emrkc_k::kMaxZc : emrkc_k::kMaxZcPipe,
                       std::max(1, std::atoi(zc)));
  return EMRKC_OK;
}

// Deterministic device norm^2 (fixed grid) of x[len].
int norm2sq(emrkc_handle* h, const double* x, int64_t len, double* out) {
  const int nb = emrkc_k::power_blocks();
  CK(h, emrkc_k::launch_norm2_partial(x, len, h->d_red, nb, h->stream));
  CK(h, emrkc_k::launch_sum_partials(h->d_red, nb, h->d_red + nb, h->stream));
  CK(h, cudaMemcpyAsync(out, h->d_red + nb, sizeof(double),
                        cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return EMRKC_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* emrkc_version(void) { return "emrkc-b200 1 (sm_100a)"; }

const char* emrkc_global_error(void) { return g_global_err.c_str(); }

int emrkc_get_stages(double dt, double rho, double epsilon, int32_t* s,
                     double* ell, double* beta) {
  int32_t s_;
  double l_, b_;
  const int rc = stages(dt, rho, epsilon, &s_, &l_, &b_);
  if (rc) return rc;
  if (s) *s = s_;
  if (ell) *ell = l_;
  if (beta) *beta = b_;
  return EMRKC_OK;
}

int emrkc_rkc_coeffs(int32_t s, double epsilon, double* omega0,
                     double* omega1, double* b, double* mu, double* nu,
                     double* kappa, double* c) {
  Coeffs k;
  const int rc = coeffs(s, epsilon, &k);
  if (rc) return rc;
  if (omega0) *omega0 = k.omega0;
  if (omega1) *omega1 = k.omega1;
  for (int j = 0; j <= s; ++j) {
    if (b) b[j] = k.b[j];
    if (mu) mu[j] = k.mu[j];
    if (nu) nu[j] = k.nu[j];
    if (kappa) kappa[j] = k.kappa[j];
    if (c) c[j] = k.c[j];
  }
  return EMRKC_OK;
}

int emrkc_plan_step(double dt, double rho_F, double rho_S, double epsilon,
                    emrkc_step_report* plan) {
  if (!plan) return set_global(EMRKC_EINVAL, "null report");
  Plan p;
  const int rc = make_plan(dt, rho_F, rho_S, epsilon, &p);
  if (rc) return rc;
  std::memset(plan, 0, sizeof(*plan));
  plan->s = p.s;
  plan->m = p.m;
  plan->eta = p.eta;
  plan->ell_s = p.ell_s;
  plan->ell_m = p.ell_m;
  plan->n_fF = static_cast<int64_t>(p.s) * p.m;
  plan->n_fS = p.s;
  plan->n_exp = p.s;
  return EMRKC_OK;
}

int emrkc_model_info(int32_t model, int32_t* n_gates, int32_t* n_aux) {
  if (model != EMRKC_MODEL_HH && model != EMRKC_MODEL_HH_AUX)
    return set_global(EMRKC_EINVAL, "unknown ionic model %d", model);
  if (n_gates) *n_gates = 3;
  // HH_AUX: the problem's n_aux (1 .. EMRKC_MAX_AUX); reported as the maximum
  if (n_aux) *n_aux = model == EMRKC_MODEL_HH ? 0 : EMRKC_MAX_AUX;
  return EMRKC_OK;
}

int emrkc_resting_state(int32_t model, double* V, double* gates) {
  if (model != EMRKC_MODEL_HH)
    return set_global(EMRKC_EINVAL, "unknown ionic model %d", model);
  // IonicModel::resting_state — bisection on [-90, -40] mV (P/src/ionic.cpp:42-77)
  double lam[3], zinf[3];
  auto steady = [&](double v) {
    hh_gate_coeffs(v, lam, zinf);
    return hh_current(v, zinf);
  };
  double lo = -90.0, hi = -40.0;
  double flo = steady(lo), fhi = steady(hi);
  if (flo * fhi > 0.0)
    return set_global(EMRKC_EINVAL, "resting_state: no sign change in [-90, -40] mV");
  for (int it = 0; it < 200 && hi - lo > 1e-14; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double fm = steady(mid);
    if (flo * fm <= 0.0) {
      hi = mid;
      fhi = fm;
    } else {
      lo = mid;
      flo = fm;
    }
  }
  const double v = 0.5 * (lo + hi);
  hh_gate_coeffs(v, lam, zinf);
  if (V) *V = v;
  if (gates)
    for (int g = 0; g < 3; ++g) gates[g] = zinf[g];
  return EMRKC_OK;
}

int64_t emrkc_state_len(const emrkc_problem* p, const emrkc_partition* part) {
  if (validate(p)) return -1;
  int64_t nn = nodes_of(p);
  if (part) {
    const int za = p->dim - 1;
    nn = nn / p->n[za] * (part->z_end - part->z_begin);
  }
  return fields_of(p) * nn;
}

int emrkc_initial_state(const emrkc_problem* p, double* y, int64_t len) {
  int rc = validate(p);
  if (rc) return rc;
  if (!y || len != fields_of(p) * nodes_of(p))
    return set_global(EMRKC_EINVAL, "initial_state: need the global state length");
  double V = 0.0, z[3];
  if ((rc = emrkc_resting_state(EMRKC_MODEL_HH, &V, z))) return rc;
  const int64_t nn = nodes_of(p);
  std::fill(y, y + nn, V);
  for (int g = 0; g < 3; ++g) std::fill(y + (1 + g) * nn, y + (2 + g) * nn, z[g]);
  for (int a = 0; a < fields_of(p) - 4; ++a)  // HHAux::resting_state (include/emrkc.h)
    std::fill(y + (4 + a) * nn, y + (5 + a) * nn, aux_s1(a) * V + aux_s0(a));
  return EMRKC_OK;
}

int emrkc_partition_slab(int64_t n_z, int32_t nranks, int32_t rank,
                         emrkc_partition* out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || n_z < nranks)
    return set_global(EMRKC_EINVAL, "partition: need 0 <= rank < nranks <= n_z");
  const int64_t base = n_z / nranks, rem = n_z % nranks;
  out->z_begin = rank * base + std::min<int64_t>(rank, rem);
  out->z_end = out->z_begin + base + (rank < rem ? 1 : 0);
  return EMRKC_OK;
}

int emrkc_create(const emrkc_problem* p, int32_t device,
                 const emrkc_partition* part, emrkc_handle** out) {
  if (!out) return set_global(EMRKC_EINVAL, "null output handle");
  *out = nullptr;
  int rc = validate(p);
  if (rc) return rc;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return set_global(EMRKC_ECUDA, "no CUDA device available (%s); there is no CPU fallback",
                      cudaGetErrorString(e));
  if (device < 0 || device >= ndev)
    return set_global(EMRKC_EINVAL, "device %d out of range (%d devices)", device, ndev);
  const int za = p->dim - 1;
  int64_t zb = 0, ze = p->n[za];
  if (part) {
    zb = part->z_begin;
    ze = part->z_end;
    if (zb < 0 || ze > p->n[za] || ze <= zb)
      return set_global(EMRKC_EINVAL, "partition: bad slab [%lld, %lld)",
                        (long long)zb, (long long)ze);
    if (p->dim == 1 && (zb != 0 || ze != p->n[0]))
      return set_global(EMRKC_EINVAL, "partition: 1-D grids are not partitioned");
  }
  auto* h = new emrkc_handle();
  h->p = *p;
  h->device = device;
  h->z_begin = zb;
  h->z_end = ze;
  h->partitioned = (zb != 0 || ze != p->n[za]);
  Geom& g = h->geom;
  g.dim = p->dim;
  g.n0 = static_cast<int>(p->n[0]);
  g.n1 = static_cast<int>(p->n[1]);
  g.n2 = static_cast<int>(p->n[2]);
  g.nzg = static_cast<int>(p->n[za]);
  g.nzl = static_cast<int>(ze - zb);
  g.zoff = static_cast<int>(zb);
  if (za == 0) g.n0 = g.nzl;
  if (za == 1) g.n1 = g.nzl;
  if (za == 2) g.n2 = g.nzl;
  g.plane = 1;
  for (int a = 0; a < za; ++a) g.plane *= p->n[a];
  g.nn = g.plane * g.nzl;
  for (int a = 0; a < 3; ++a)
    g.w[a] = (a < p->dim) ? p->sigma[a] / (p->chi * p->C_m * p->dx[a] * p->dx[a])
                          : 0.0;
  g.wc = -2.0 * (g.w[0] + g.w[1] + g.w[2]);
  g.Cm = p->C_m;
  g.inv_Cm = 1.0 / p->C_m;
  for (int a = 0; a < 3; ++a) {
    if (a < p->dim) {
      stim_range(p, a, &g.st_lo[a], &g.st_hi[a]);
    } else {
      g.st_lo[a] = 0;
      g.st_hi[a] = 0;
    }
  }
  g.naux = fields_of(p) - 4;
  g.nf = fields_of(p);
  h->nn = g.nn;
  h->len = static_cast<int64_t>(g.nf) * g.nn;
  if ((rc = init_handle(h))) {
    g_global_err = h->err;
    emrkc_destroy(h);
    return rc;
  }
  *out = h;
  return EMRKC_OK;
}

void emrkc_destroy(emrkc_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (auto& b : h->buf)
    if (b) cudaFree(b);
  if (h->fs) cudaFree(h->fs);
  if (h->ye) cudaFree(h->ye);
  for (auto& u : h->u)
    if (u) cudaFree(u);
  for (auto& pe : h->peer)
    if (pe.ipc && pe.arena) cudaIpcCloseMemHandle(pe.arena);
  if (h->arena) cudaFree(h->arena);
  if (h->ckpt) cudaFree(h->ckpt);
  if (h->res_v) cudaFree(h->res_v);
  if (h->res_stim) cudaFree(h->res_stim);
  if (h->d_event) cudaFree(h->d_event);
  if (h->d_slots) cudaFree(h->d_slots);
  if (h->d_coef) cudaFree(h->d_coef);
  if (h->d_red) cudaFree(h->d_red);
  if (h->d_rel) cudaFree(h->d_rel);
  if (h->fu_xch) cudaFree(h->fu_xch);
  for (auto e : h->zp_ev)
    if (e) cudaEventDestroy(e);
  if (h->zp_join) cudaEventDestroy(h->zp_join);
  if (h->s_aux) cudaStreamDestroy(h->s_aux);
  for (auto p : {h->sp_v[0], h->sp_v[1], h->sp_fy})
    if (p) cudaFree(p);
  if (h->fu_flags) cudaFree(h->fu_flags);
  for (auto& u : h->mr_u)
    if (u) cudaFree(u);
  if (h->mr_fs) cudaFree(h->mr_fs);
  if (h->cg_v) cudaFree(h->cg_v);
  if (h->cg_part) cudaFree(h->cg_part);
  if (h->cg_s) cudaFree(h->cg_s);
  if (h->cg_h) cudaFreeHost(h->cg_h);
  if (h->guard_d) cudaFree(h->guard_d);
  if (h->d_tmp) cudaFree(h->d_tmp);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  for (auto e : h->ev_in) cudaEventDestroy(e);
  for (auto e : h->ev_k) cudaEventDestroy(e);
  if (h->h_event) cudaFreeHost(h->h_event);
  if (h->s_in) cudaStreamDestroy(h->s_in);
  if (h->s_out) cudaStreamDestroy(h->s_out);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

const char* emrkc_last_error(const emrkc_handle* h) {
  return h ? h->err.c_str() : g_global_err.c_str();
}

int64_t emrkc_local_len(const emrkc_handle* h) { return h ? h->len : -1; }

int emrkc_set_state(emrkc_handle* h, const double* y, int64_t len) {
  if (!h || !y) return set_global(EMRKC_EINVAL, "null argument");
  if (len != h->len)
    return set_err(h, EMRKC_EINVAL, "MonodomainOperator: state size mismatch (%lld != %lld)",
                   (long long)len, (long long)h->len);
  int rc = use_device(h);
  if (rc) return rc;
  if ((rc = ensure_buffers(h, std::max(2, h->nbuf)))) return rc;
  CK(h, cudaMemcpyAsync(h->buf[h->cur], y, sizeof(double) * len,
                        cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  h->has_state = true;
  return EMRKC_OK;
}

int emrkc_get_state(emrkc_handle* h, double* y, int64_t len) {
  if (!h || !y) return set_global(EMRKC_EINVAL, "null argument");
  if (!h->has_state) return set_err(h, EMRKC_ESTATE, "no state uploaded");
  if (len != h->len)
    return set_err(h, EMRKC_EINVAL, "state size mismatch");
  int rc = use_device(h);
  if (rc) return rc;
  CK(h, cudaMemcpyAsync(y, h->buf[h->cur], sizeof(double) * len,
                        cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return EMRKC_OK;
}

int emrkc_rel_l2_error(emrkc_handle* h, int32_t block, const double* ref, int32_t ref_on_device,
                       double* out) {
  if (!h || !ref || !out) return set_global(EMRKC_EINVAL, "null argument");
  if (h->partitioned) return set_err(h, EMRKC_EINVAL, "rel_l2_error: whole-grid handles only");
  if (block < 0 || block > 3) return set_err(h, EMRKC_EINVAL, "rel_l2_error: block must be 0..3");
  if (!h->has_state) return set_err(h, EMRKC_ESTATE, "no state uploaded");
  int rc = use_device(h);
  if (rc) return rc;
  const int nb = 512;
  if (!h->d_rel) CK(h, cudaMalloc(&h->d_rel, sizeof(double) * (2 * nb + 2)));
  const double* b = ref;
  if (!ref_on_device) {
    if (!h->d_tmp) CK(h, cudaMalloc(&h->d_tmp, sizeof(double) * h->nn));
    CK(h, cudaMemcpyAsync(h->d_tmp, ref, sizeof(double) * h->nn, cudaMemcpyHostToDevice,
                          h->stream));
    b = h->d_tmp;
  }
  CK(h, emrkc_k::launch_rel_l2(h->geom, h->buf[h->cur] + block * h->nn, b, h->d_rel, nb,
                               h->d_rel + 2 * nb, h->stream));
  double s[2] = {0.0, 0.0};
  CK(h, cudaMemcpyAsync(s, h->d_rel + 2 * nb, sizeof(s), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  // l2_norm(u) = sqrt(cell * sum w u^2)  (P/src/monodomain.cpp:92-99)
  double cell = 1.0;
  for (int a = 0; a < h->p.dim; ++a) cell *= h->p.dx[a];
  const double nbn = std::sqrt(cell * s[1]);
  if (nbn == 0.0) return set_err(h, EMRKC_EINVAL, "rel_l2_error: ||b|| is zero");
  *out = std::sqrt(cell * s[0]) / nbn;
  return EMRKC_OK;
}

int emrkc_state_device_ptr(emrkc_handle* h, double** dptr) {
  if (!h || !dptr) return set_global(EMRKC_EINVAL, "null argument");
  if (!h->has_state) return set_err(h, EMRKC_ESTATE, "no state uploaded");
  *dptr = h->buf[h->cur];
  return EMRKC_OK;
}

int emrkc_synchronize(emrkc_handle* h) {
  if (!h) return set_global(EMRKC_EINVAL, "null handle");
  int rc = use_device(h);
  if (rc) return rc;
  CK(h, cudaStreamSynchronize(h->stream));
  return EMRKC_OK;
}

namespace {
// emrkc_eval_rhs / emrkc_estimate_rho selector -> kernel code: F / S, and for
// the mRKC split f_F / f_S with gate rows (mask in bits 4..6).
int rhs_code(const emrkc_handle* h, int32_t which, int* code) {
  switch (which) {
    case EMRKC_RHS_F: *code = 0; return EMRKC_OK;
    case EMRKC_RHS_S: *code = 1; return EMRKC_OK;
    case EMRKC_RHS_F_GATES: *code = 0 | ((h->stiff & 7) << 4); return EMRKC_OK;
    case EMRKC_RHS_S_GATES: *code = 1 | ((~h->stiff & 7) << 4); return EMRKC_OK;
    default: return EMRKC_EINVAL;
  }
}

}  // namespace

int emrkc_eval_rhs(emrkc_handle* h, int32_t which, double t, const double* y,
                   double* out, int64_t len) {
  if (!h || !y || !out) return set_global(EMRKC_EINVAL, "null argument");
  if (h->partitioned) return set_err(h, EMRKC_EINVAL, "eval_rhs: whole-grid handles only");
  if (len != h->len) return set_err(h, EMRKC_EINVAL, "MonodomainOperator: state size mismatch");
  int code = 0;
  if (rhs_code(h, which, &code)) return set_err(h, EMRKC_EINVAL, "eval_rhs: unknown rhs %d", which);
  int rc = use_device(h);
  if (rc) return rc;
  double *dy = nullptr, *dout = nullptr;
  CK(h, cudaMalloc(&dy, sizeof(double) * len));
  CK(h, cudaMalloc(&dout, sizeof(double) * len));
  CK(h, cudaMemcpyAsync(dy, y, sizeof(double) * len, cudaMemcpyHostToDevice, h->stream));
  CK(h, emrkc_k::launch_rhs(h->geom, Halo{}, code, dy, stim_rate_at(&h->p, t), dout,
                            h->stream));
  CK(h, cudaMemcpyAsync(out, dout, sizeof(double) * len, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  cudaFree(dy);
  cudaFree(dout);
  return EMRKC_OK;
}

int emrkc_exp_part(emrkc_handle* h, const double* y, double* lambda,
                   double* y_inf, int64_t len) {
  if (!h || !y || !lambda || !y_inf) return set_global(EMRKC_EINVAL, "null argument");
  if (len != h->len) return set_err(h, EMRKC_EINVAL, "MonodomainOperator: state size mismatch");
  int rc = use_device(h);
  if (rc) return rc;
  double *dy = nullptr, *dl = nullptr, *di = nullptr;
  CK(h, cudaMalloc(&dy, sizeof(double) * len));
  CK(h, cudaMalloc(&dl, sizeof(double) * len));
  CK(h, cudaMalloc(&di, sizeof(double) * len));
  CK(h, cudaMemcpyAsync(dy, y, sizeof(double) * len, cudaMemcpyHostToDevice, h->stream));
  CK(h, emrkc_k::launch_exp_part(h->geom, dy, dl, di, h->stream));
  CK(h, cudaMemcpyAsync(lambda, dl, sizeof(double) * len, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaMemcpyAsync(y_inf, di, sizeof(double) * len, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  cudaFree(dy);
  cudaFree(dl);
  cudaFree(di);
  return EMRKC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Power iteration (shared by single handles and groups)
// ---------------------------------------------------------------------------
namespace {

// seeded_direction (P/src/spectral.cpp:16-22): libstdc++ mt19937_64 +
// uniform_real_distribution(-1, 1) over the full global state.
void seeded_direction(std::vector<double>& v) {
  std::mt19937_64 rng(0x9e3779b97f4a7c15ull);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (double& x : v) x = dist(rng);
}

// Global-vector slice of a slab handle: block b, local nodes.
void scatter_slab(const emrkc_handle* h, const std::vector<double>& global,
                  int64_t global_nn, std::vector<double>& local) {
  local.resize(h->len);
  const int64_t off = h->z_begin * h->geom.plane;
  for (int b = 0; b < h->geom.nf; ++b)
    std::memcpy(local.data() + b * h->nn, global.data() + b * global_nn + off,
                sizeof(double) * h->nn);
}

struct PowerWork {
  double* v[2] = {nullptr, nullptr};
  double* fy = nullptr;
  double* gy[2] = {nullptr, nullptr};  // ghost planes of y_V (below, above)
  double* gv[2] = {nullptr, nullptr};  // ghost planes of v_V
};

int power_alloc(emrkc_handle* h, PowerWork* w) {
  CK(h, cudaSetDevice(h->device));
  CK(h, cudaMalloc(&w->v[0], sizeof(double) * h->len));
  CK(h, cudaMalloc(&w->v[1], sizeof(double) * h->len));
  CK(h, cudaMalloc(&w->fy, sizeof(double) * h->len));
  if (h->partitioned)
    for (int s = 0; s < 2; ++s) {
      CK(h, cudaMalloc(&w->gy[s], sizeof(double) * h->geom.plane));
      CK(h, cudaMalloc(&w->gv[s], sizeof(double) * h->geom.plane));
    }
  return EMRKC_OK;
}

void power_free(emrkc_handle* h, PowerWork* w) {
  cudaSetDevice(h->device);
  for (auto p : {w->v[0], w->v[1], w->fy, w->gy[0], w->gy[1], w->gv[0], w->gv[1]})
    if (p) cudaFree(p);
}

// Copy the neighbours' boundary V planes of field f (per handle) into the
// ghost buffers dst (per handle, [below, above]).
int exchange_planes(const std::vector<emrkc_handle*>& hs,
                    const std::vector<const double*>& field,
                    const std::vector<double* const*>& dst) {
  const size_t n = hs.size();
  for (size_t r = 0; r < n; ++r) {
    emrkc_handle* h = hs[r];
    const size_t bytes = sizeof(double) * h->geom.plane;
    if (r > 0) {  // below: neighbour's last plane
      emrkc_handle* nb = hs[r - 1];
      const double* src = field[r - 1] + (nb->nn - nb->geom.plane);
      CK(h, cudaMemcpyPeer(dst[r][0], h->device, src, nb->device, bytes));
    }
    if (r + 1 < n) {  // above: neighbour's first plane
      emrkc_handle* nb = hs[r + 1];
      CK(h, cudaMemcpyPeer(dst[r][1], h->device, field[r + 1], nb->device, bytes));
    }
  }
  return EMRKC_OK;
}

bool rho_serial() {
  static const bool on = [] {
    const char* e = std::getenv("EMRKC_RHO_SERIAL");
    return !(e && *e == '0');
  }();
  return on;
}

// estimate_spectral_radius (P/src/spectral.cpp:26-71) over a list of slabs
// (one whole-grid handle is the common case). Norms are sums of per-slab
// deterministic device reductions.
int power_iteration(const std::vector<emrkc_handle*>& hs, int which, double t,
                    const double* v0_global, double rho0, emrkc_rho_result* out,
                    double* v_out_global) {
  const size_t n = hs.size();
  emrkc_handle* h0 = hs[0];
  const emrkc_problem& p = h0->p;
  const int64_t gnn = nodes_of(&p);
  const int64_t glen = static_cast<int64_t>(h0->geom.nf) * gnn;
  for (auto* h : hs)
    if (!h->has_state) return set_err(h, EMRKC_ESTATE, "no state uploaded");
  std::vector<double> v0(glen);
  if (v0_global)
    std::memcpy(v0.data(), v0_global, sizeof(double) * glen);
  else
    seeded_direction(v0);
  std::vector<PowerWork> w(n);
  int rc = EMRKC_OK;
  int a = 0;
  const double stim = stim_rate_at(&p, t);
  const double kEps = 1e-8, kTol = 1e-2;
  const int kMaxIters = 50;
  auto cleanup = [&]() {
    for (size_t r = 0; r < n; ++r) power_free(hs[r], &w[r]);
  };
  // ||x||^2 in the reference's serial order (P/src/spectral.cpp:10-14) over
  // the global vector: SoA block by block, slabs in z order within a block,
  // the running sum chained from piece to piece. Bit-identical to the
  // reference, so q, z, f(z) - f(y) and rho are too (EMRKC_RHO_SERIAL=0:
  // the deterministic parallel reduction instead, ~1e-12 relative).
  auto sum_norm2 = [&](auto field_of) -> double {
    double tot = 0.0;
    if (!rho_serial()) {
      for (size_t r = 0; r < n; ++r) {
        double part = 0.0;
        rc = norm2sq(hs[r], field_of(r), hs[r]->len, &part);
        if (rc) return 0.0;
        tot += part;
      }
      return tot;
    }
    for (int b = 0; b < h0->geom.nf; ++b)
      for (size_t r = 0; r < n; ++r) {
        emrkc_handle* h = hs[r];
        cudaSetDevice(h->device);
        cudaError_t e = emrkc_k::launch_sumsq_serial(field_of(r) + b * h->nn, h->nn, tot,
                                                     h->d_red, h->stream);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(&tot, h->d_red, sizeof(double), cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) {
          rc = set_err(h, EMRKC_ECUDA, "power iteration: %s", cudaGetErrorString(e));
          return 0.0;
        }
      }
    return tot;
  };
  std::vector<const double*> ys(n), vs(n);
  std::vector<double* const*> gys(n), gvs(n);
  double nv_cur, ny, delta, rho = rho0, rho_old = 0.0;
  int it = 0;
  out->safety = 1.05;
  out->converged = 1;
  for (size_t r = 0; r < n; ++r) {
    if ((rc = power_alloc(hs[r], &w[r]))) goto fail;
    std::vector<double> local;
    scatter_slab(hs[r], v0, gnn, local);
    cudaError_t e = cudaMemcpy(w[r].v[0], local.data(), sizeof(double) * hs[r]->len,
                               cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      rc = set_err(hs[r], EMRKC_ECUDA, "%s", cudaGetErrorString(e));
      goto fail;
    }
    ys[r] = hs[r]->buf[hs[r]->cur];
    gys[r] = w[r].gy;
    gvs[r] = w[r].gv;
  }
  nv_cur = std::sqrt(sum_norm2([&](size_t r) { return w[r].v[0]; }));
  if (rc) goto fail;
  if (nv_cur == 0.0) {
    rc = set_err(h0, EMRKC_EINVAL, "estimate_spectral_radius: v0 must be nonzero");
    goto fail;
  }
  ny = std::sqrt(sum_norm2([&](size_t r) { return ys[r]; }));
  if (rc) goto fail;
  delta = std::max(ny, kEps) * kEps;
  if (n > 1 && (rc = exchange_planes(hs, ys, gys))) goto fail;
  for (size_t r = 0; r < n; ++r) {
    emrkc_handle* h = hs[r];
    Halo hh{};
    hh.lo = w[r].gy[0];
    hh.hi = w[r].gy[1];
    if (r == 0) hh.lo = nullptr;
    if (r + 1 == n) hh.hi = nullptr;
    cudaSetDevice(h->device);
    cudaError_t e = emrkc_k::launch_rhs(h->geom, hh, which, ys[r], stim, w[r].fy, h->stream);
    if (e != cudaSuccess) {
      rc = set_err(h, EMRKC_ECUDA, "%s", cudaGetErrorString(e));
      goto fail;
    }
  }
  while (it == 0 || std::abs(rho - rho_old) >= kTol * rho) {
    if (it >= kMaxIters) {
      out->converged = 0;
      break;
    }
    rho_old = rho;
    const double q = delta / nv_cur;
    for (size_t r = 0; r < n; ++r) vs[r] = w[r].v[a];
    if (n > 1 && (rc = exchange_planes(hs, vs, gvs))) goto fail;
    double tot = 0.0;
    for (size_t r = 0; r < n; ++r) {
      emrkc_handle* h = hs[r];
      cudaSetDevice(h->device);
      const int nb = emrkc_k::power_blocks();
      cudaError_t e = emrkc_k::launch_power(
          h->geom, which, ys[r], w[r].v[a], q, w[r].fy, stim, w[r].v[1 - a],
          r > 0 ? w[r].gy[0] : nullptr, r + 1 < n ? w[r].gy[1] : nullptr,
          r > 0 ? w[r].gv[0] : nullptr, r + 1 < n ? w[r].gv[1] : nullptr,
          h->d_red, nb, h->stream);
      if (e == cudaSuccess)
        e = emrkc_k::launch_sum_partials(h->d_red, nb, h->d_red + nb, h->stream);
      double part = 0.0;
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(&part, h->d_red + nb, sizeof(double),
                            cudaMemcpyDeviceToHost, h->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
      if (e != cudaSuccess) {
        rc = set_err(h, EMRKC_ECUDA, "power iteration: %s", cudaGetErrorString(e));
        goto fail;
      }
      tot += part;
    }
    if (rho_serial()) {
      const int an = 1 - a;
      tot = sum_norm2([&](size_t r) { return w[r].v[an]; });
      if (rc) goto fail;
    }
    a = 1 - a;
    const double nv = std::sqrt(tot);
    if (nv < 1e-300) {
      out->rho = 0.0;
      out->iterations = it + 1;
      goto vout;
    }
    rho = nv / delta;
    nv_cur = nv;
    ++it;
  }
  out->rho = rho * out->safety;
  out->iterations = it;
vout:
  if (v_out_global) {
    for (size_t r = 0; r < n; ++r) {
      emrkc_handle* h = hs[r];
      std::vector<double> local(h->len);
      cudaSetDevice(h->device);
      cudaMemcpy(local.data(), w[r].v[a], sizeof(double) * h->len, cudaMemcpyDeviceToHost);
      const int64_t off = h->z_begin * h->geom.plane;
      for (int b = 0; b < h->geom.nf; ++b)
        std::memcpy(v_out_global + b * gnn + off, local.data() + b * h->nn,
                    sizeof(double) * h->nn);
    }
  }
fail:
  cleanup();
  return rc;
}

// ---------------------------------------------------------------------------
// Run loop over a list of slabs in lockstep (one handle: the plain run).
// ---------------------------------------------------------------------------
// EmrkcVariant -> method (P/include/mrkc/multirate.hpp:37-40).
int variant_method(int32_t variant, int* method) {
  if (variant == EMRKC_VARIANT_STANDARD) *method = kMethodEmrkc;
  else if (variant == EMRKC_VARIANT_PROGRESSIVE) *method = kMethodEmrkcProgressive;
  else return EMRKC_EINVAL;
  return EMRKC_OK;
}

// Whole-run resident kernel (k_resident): small whole-grid runs with
// s = m = 1 on the fast kernels (EMRKC_RESIDENT=0 disables).
bool resident_ok(const emrkc_handle* h, int64_t nsteps) {
  static const bool on = [] {
    const char* e = std::getenv("EMRKC_RESIDENT");
    return !(e && *e == '0');
  }();
  const Plan& pl = h->plan;
  return on && h->fast && !h->partitioned && nsteps >= 2 && nsteps <= 10000000 &&
         h->geom.naux == 0 &&
         pl.s == 1 && pl.m == 1 &&
         pl.method != kMethodMrkc && (h->geom.dim == 2 || h->geom.dim == 3) &&
         h->geom.nn <= emrkc_k::resident_capacity(h->geom.dim);
}

// One cooperative launch for steps step0 .. step0 + nsteps - 1; the run's
// final state lands in buffer *out_idx. The abort word and the per-step
// gate-range slots are the per-step kernels' (decode_event, fold).
int run_resident(emrkc_handle* h, int64_t step0, int64_t nsteps, int* out_idx) {
  const Plan& pl = h->plan;
  int rc = ensure_buffers(h, std::max(2, h->nbuf));
  if (rc) return rc;
  const int in = h->cur, out = (in + 1) % h->nbuf;
  if (!h->res_v) CK(h, cudaMalloc(&h->res_v, sizeof(double) * (2 * h->nn + 2)));
  unsigned* bar = reinterpret_cast<unsigned*>(h->res_v + 2 * h->nn);
  CK(h, cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), h->stream));
  if (h->res_stim_n < nsteps) {
    if (h->res_stim) cudaFree(h->res_stim);
    h->res_stim = nullptr;
    CK(h, cudaMalloc(&h->res_stim, sizeof(double) * nsteps));
    h->res_stim_n = nsteps;
  }
  std::vector<double> stim(nsteps);
  for (int64_t r = 0; r < nsteps; ++r)  // stage time t = step dt (simulate.cpp:177)
    stim[r] = stim_rate_at(&h->p, static_cast<double>(step0 + r) * pl.dt);
  CK(h, cudaMemcpyAsync(h->res_stim, stim.data(), sizeof(double) * nsteps,
                        cudaMemcpyHostToDevice, h->stream));
  emrkc_k::ResidentArgs ra{};
  emrkc_k::FastArgs& f = ra.f;  // launch_level's j = k = 1 arguments
  const double cG = pl.mudt[1] / pl.eta;
  f.eta = pl.eta;
  f.cG = cG * pl.gate_c;
  f.cV = cG * pl.in_mueta[1];
  f.mue1 = pl.in_mueta[1];
  f.exex = pl.exex;
  fast_window(pl.eta, &f.vmid, &f.vfast);
  f.j = 1;
  f.m = pl.m;
  f.s = pl.s;
  f.last = 1;
  f.z_lo = 0;
  f.z_hi = h->geom.nzl;
  f.event = h->d_event;
  ra.y_in = h->buf[in];
  ra.y_out = h->buf[out];
  ra.vbuf = h->res_v;
  ra.stim = h->res_stim;
  ra.nsteps = nsteps;
  ra.stride = static_cast<unsigned long long>(pl.s) * (pl.m + 1) + 2;  // begin_step's
  ra.slots = h->d_slots;
  ra.bar = bar;
  const cudaError_t e = emrkc_k::launch_resident(h->geom, ra, h->stream);
  if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorInvalidValue) {
    cudaGetLastError();  // not co-resident here (e.g. a shared GPU): per-step launches
    return -1;
  }
  CK(h, e);
  *out_idx = out;
  return EMRKC_OK;
}

int run_slabs(const std::vector<emrkc_handle*>& hs, int64_t step0,
              int64_t nsteps, double dt, double eps, double rho_F,
              double rho_S, emrkc_run_result* res, bool single_step,
              emrkc_step_report* rep, int64_t flush_bytes = 0,
              double* launch_ms = nullptr, int64_t launch_ms_len = 0,
              bool lockstep = false) {
  const size_t n = hs.size();
  int rc;
  const bool dist = dist_linked(hs[0]);
  if (dist)
    for (auto* h : hs) {
      if (!h->fast)
        return set_err(h, EMRKC_EINVAL, "distributed runs need the fast kernels (EMRKC_FAST=1)");
      if ((h->z_begin > 0 && !h->peer[0].linked) ||
          (h->z_end < h->p.n[h->p.dim - 1] && !h->peer[1].linked))
        return set_err(h, EMRKC_ESTATE, "dist_run: neighbour not imported");
    }
  for (auto* h : hs) {
    if (!h->has_state) return set_err(h, EMRKC_ESTATE, "no state uploaded");
    if ((rc = use_device(h))) return rc;
    if ((rc = upload_plan(h, dt, rho_F, rho_S, eps))) return rc;
    if ((rc = ensure_slots(h, static_cast<size_t>(nsteps)))) return rc;
    CK(h, cudaMemcpyAsync(h->d_event, &kNoEvent, sizeof(kNoEvent),
                          cudaMemcpyHostToDevice, h->stream));
    CK(h, emrkc_k::launch_fill_u64(h->d_slots, 2 * (nsteps + 1), 0, h->stream));
    // min slots start at ~0, max slots at 0
    std::vector<unsigned long long> init(2 * (nsteps + 1));
    for (size_t k = 0; k < init.size(); k += 2) {
      init[k] = kNoEvent;
      init[k + 1] = 0ull;
    }
    CK(h, cudaMemcpyAsync(h->d_slots, init.data(), sizeof(unsigned long long) * init.size(),
                          cudaMemcpyHostToDevice, h->stream));
    CK(h, emrkc_k::launch_gate_range(h->geom, h->buf[h->cur],
                                     h->d_slots + 2 * nsteps, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    h->slot_init = single_step ? nullptr : h->d_slots + 2 * nsteps;
  }
  struct SlotReset {  // the slot chain only holds inside this run
    const std::vector<emrkc_handle*>& v;
    ~SlotReset() {
      for (auto* q : v) q->slot_init = nullptr;
    }
  } slot_reset{hs};
  const Plan& pl = hs[0]->plan;
  // Initial ghost planes of the current state (level L0 slot).
  if (n > 1) {
    const long long L0 = hs[0]->level;
    for (auto* h : hs)
      if (h->level != L0) return set_err(h, EMRKC_ESTATE, "group handles out of step");
    std::vector<const double*> f(n);
    std::vector<double* const*> dst(n);
    std::vector<std::array<double*, 2>> slots(n);
    for (size_t r = 0; r < n; ++r) {
      f[r] = hs[r]->buf[hs[r]->cur];
      slots[r] = {hs[r]->ghost[0][L0 & 1], hs[r]->ghost[1][L0 & 1]};
      dst[r] = slots[r].data();
    }
    if (!dist) {
      if ((rc = exchange_planes(hs, f, dst))) return rc;
      for (auto* h : hs) CK(h, cudaDeviceSynchronize());
    }
  }
  if (dist) {
    // checkpoint for emrkc_dist_replay, then the prime level: every slab
    // pushes its boundary V planes into the neighbours' current ghost slot
    cudaEvent_t prev = nullptr;
    for (auto* h : hs) {
      CK(h, cudaSetDevice(h->device));
      if (!h->ckpt) CK(h, cudaMalloc(&h->ckpt, sizeof(double) * h->len));
      CK(h, cudaMemcpyAsync(h->ckpt, h->buf[h->cur], sizeof(double) * h->len,
                            cudaMemcpyDeviceToDevice, h->stream));
      if (lockstep && prev) CK(h, cudaStreamWaitEvent(h->stream, prev, 0));
      Halo hp{};
      const int ws = static_cast<int>(h->level & 1);
      if (h->peer[0].linked) {
        hp.put_lo = h->peer[0].ghost[ws];
        hp.sig_lo = h->peer[0].cnt;
      }
      if (h->peer[1].linked) {
        hp.put_hi = h->peer[1].ghost[ws];
        hp.sig_hi = h->peer[1].cnt;
      }
      CK(h, emrkc_k::launch_halo_prime(h->geom, hp, h->buf[h->cur], h->stream));
      dist_account(h, emrkc_k::halo_signals_prime(h->geom));
      if (h->level_hook) {
        CK(h, cudaStreamSynchronize(h->stream));
        h->level_hook(h->level_ctx);
      }
      CK(h, cudaEventRecord(h->ev1, h->stream));
      prev = h->ev1;
    }
  }
  std::vector<std::vector<int>> in_idx(n, std::vector<int>(nsteps + 1));
  for (auto* h : hs) {
    CK(h, cudaSetDevice(h->device));
    CK(h, cudaEventRecord(h->ev0, h->stream));
  }
  std::vector<cudaEvent_t> tev;
  int resident_out = 0;
  if (n == 1 && launch_ms) {
    // benchmark form: flush L2 before each step, one event pair per launch
    emrkc_handle* h = hs[0];
    const int64_t per = static_cast<int64_t>(pl.s) * pl.m;
    if (launch_ms_len < nsteps * per)
      return set_err(h, EMRKC_EINVAL, "run_timed: launch_ms needs %lld entries",
                     (long long)(nsteps * per));
    // L2 flush between steps: write a buffer larger than L2, then read a
    // second one so the dirty lines are written back outside the timed
    // pairs (L2 left cold and clean)
    void* scratch = nullptr;
    void* scratch_rd = nullptr;
    if (flush_bytes > 0) {
      CK(h, cudaMalloc(&scratch, flush_bytes));
      CK(h, cudaMalloc(&scratch_rd, flush_bytes));
      CK(h, cudaMemset(scratch_rd, 0, flush_bytes));
    }
    tev.resize(2 * nsteps * per);
    for (auto& e : tev) CK(h, cudaEventCreate(&e));
    int64_t li = 0;
    const bool xs = use_xstep(h, pl, nsteps);
    StepCtx xc;
    if (xs && (rc = ensure_buffers(h, 3))) return rc;
    for (int64_t r = 0; r < nsteps; ++r) {
      const double t = static_cast<double>(step0 + r) * dt;
      if (!xs || r == 0) in_idx[0][r] = h->cur;
      if (xs && r + 1 < nsteps) in_idx[0][r + 1] = (h->cur + 1) % h->nbuf;
      if (scratch) {
        CK(h, cudaMemsetAsync(scratch, static_cast<int>(r & 0xff), flush_bytes, h->stream));
        CK(h, emrkc_k::launch_norm2_partial(static_cast<const double*>(scratch_rd),
                                            flush_bytes / 8, h->d_red,
                                            emrkc_k::power_blocks(), h->stream));
      }
      if (use_zpipe(h, pl)) {
        // two streams overlap: one event pair around the whole step (first
        // entry), the other entries of the step 0
        CK(h, cudaEventRecord(tev[2 * li], h->stream));
        int outi = 0;
        if ((rc = enqueue_step_zpipe(h, t, r, h->d_slots + 2 * r, &outi))) return rc;
        CK(h, cudaEventRecord(tev[2 * li + 1], h->stream));
        for (int64_t q = 1; q < per; ++q) {
          CK(h, cudaEventRecord(tev[2 * (li + q)], h->stream));
          CK(h, cudaEventRecord(tev[2 * (li + q) + 1], h->stream));
        }
        li += per;
        h->cur = outi;
        continue;
      }
      if (xs) {
        // entry 2r: the node level (a launch of its own only for r = 0),
        // entry 2r + 1: inner(r) fused with node(r + 1), or inner(r) alone
        // for the last step
        if (r == 0) {
          begin_step(h, t, 0, h->d_slots, &xc);
          CK(h, cudaEventRecord(tev[0], h->stream));
          if ((rc = launch_level(h, &xc, 1, 1))) return rc;
          CK(h, cudaEventRecord(tev[1], h->stream));
        } else {
          CK(h, cudaEventRecord(tev[2 * li], h->stream));
          CK(h, cudaEventRecord(tev[2 * li + 1], h->stream));
        }
        ++li;
        CK(h, cudaEventRecord(tev[2 * li], h->stream));
        if (r + 1 < nsteps) {
          h->cur = end_step(h, &xc);
          StepCtx cn;
          begin_step(h, static_cast<double>(step0 + r + 1) * dt, r + 1,
                     h->d_slots + 2 * (r + 1), &cn);
          if ((rc = launch_xstep(h, &xc, &cn))) return rc;
          xc = cn;
        } else {
          if ((rc = launch_level(h, &xc, 1, 2))) return rc;
          h->cur = end_step(h, &xc);
        }
        CK(h, cudaEventRecord(tev[2 * li + 1], h->stream));
        ++li;
        continue;
      }
      StepCtx c;
      begin_step(h, t, r, h->d_slots + 2 * r, &c);
      for (int j = 1; j <= pl.s; ++j)
        for (int k = 1; k <= pl.m; ++k, ++li) {
          CK(h, cudaEventRecord(tev[2 * li], h->stream));
          if ((rc = launch_level(h, &c, j, k))) return rc;
          CK(h, cudaEventRecord(tev[2 * li + 1], h->stream));
        }
      h->cur = end_step(h, &c);
    }
    CK(h, cudaStreamSynchronize(h->stream));
    double tot = 0.0;
    for (int64_t i = 0; i < nsteps * per; ++i) {
      float f = 0.0f;
      CK(h, cudaEventElapsedTime(&f, tev[2 * i], tev[2 * i + 1]));
      launch_ms[i] = f;
      tot += f;
    }
    for (auto& e : tev) cudaEventDestroy(e);
    if (scratch) cudaFree(scratch);
    if (scratch_rd) cudaFree(scratch_rd);
    if (res) res->device_ms = tot;  // overwritten below, restored after
  } else if (n == 1 && !single_step && resident_ok(hs[0], nsteps) &&
             (rc = run_resident(hs[0], step0, nsteps, &resident_out)) >= 0) {
    if (rc) return rc;
    emrkc_handle* h = hs[0];
    for (int64_t r = 0; r < nsteps; ++r) in_idx[0][r] = resident_out;  // rollback is in-kernel
    h->cur = resident_out;
  } else if (n == 1 && use_xstep(hs[0], pl, nsteps)) {
    // node(0), then inner(r) + node(r + 1) per launch, then inner(nsteps - 1)
    emrkc_handle* h = hs[0];
    if ((rc = ensure_buffers(h, 3))) return rc;
    StepCtx c, cn;
    in_idx[0][0] = h->cur;
    begin_step(h, static_cast<double>(step0) * dt, 0, h->d_slots, &c);
    if ((rc = launch_level(h, &c, 1, 1))) return rc;
    for (int64_t r = 0; r < nsteps; ++r) {
      if (r + 1 < nsteps) {
        h->cur = end_step(h, &c);
        in_idx[0][r + 1] = h->cur;
        begin_step(h, static_cast<double>(step0 + r + 1) * dt, r + 1, h->d_slots + 2 * (r + 1),
                   &cn);
        if ((rc = launch_xstep(h, &c, &cn))) return rc;
        c = cn;
      } else {
        if ((rc = launch_level(h, &c, 1, 2))) return rc;
        h->cur = end_step(h, &c);
      }
    }
  } else if (n == 1) {
    emrkc_handle* h = hs[0];
    for (int64_t r = 0; r < nsteps; ++r) {
      const double t = static_cast<double>(step0 + r) * dt;  // simulate.cpp:177
      in_idx[0][r] = h->cur;
      int outi = 0;
      if ((rc = enqueue_step(h, t, r, h->d_slots + 2 * r, &outi))) return rc;
      h->cur = outi;
    }
  } else {
    // Lockstep over slabs: after every level each slab waits for its
    // neighbours' kernels of that level (their peer stores fill its ghost
    // planes); after every step all slabs meet and fold the abort words so
    // that every slab freezes on the same step.
    std::vector<StepCtx> c(n);
    std::vector<unsigned long long*> evs(n);
    for (size_t q = 0; q < n; ++q) evs[q] = hs[q]->d_event;
    auto sync_neighbours = [&]() -> int {
      for (size_t q = 0; q < n; ++q) {
        CK(hs[q], cudaSetDevice(hs[q]->device));
        CK(hs[q], cudaEventRecord(hs[q]->ev1, hs[q]->stream));
      }
      for (size_t q = 0; q < n; ++q) {
        CK(hs[q], cudaSetDevice(hs[q]->device));
        if (q > 0) CK(hs[q], cudaStreamWaitEvent(hs[q]->stream, hs[q - 1]->ev1, 0));
        if (q + 1 < n) CK(hs[q], cudaStreamWaitEvent(hs[q]->stream, hs[q + 1]->ev1, 0));
      }
      return EMRKC_OK;
    };
    for (int64_t r = 0; r < nsteps; ++r) {
      const double t = static_cast<double>(step0 + r) * dt;  // simulate.cpp:177
      for (size_t q = 0; q < n; ++q) {
        in_idx[q][r] = hs[q]->cur;
        begin_step(hs[q], t, r, hs[q]->d_slots + 2 * r, &c[q]);
      }
      for (int j = 1; j <= pl.s; ++j)
        for (int k = 1; k <= pl.m; ++k) {
          for (size_t q = 0; q < n; ++q) {
            CK(hs[q], cudaSetDevice(hs[q]->device));
            if (lockstep) {
              // serialise every launch: each device-side wait is already
              // satisfied when its kernel starts (test driver on one GPU)
              const size_t prevq = q == 0 ? n - 1 : q - 1;
              CK(hs[q], cudaStreamWaitEvent(hs[q]->stream, hs[prevq]->ev1, 0));
            }
            if ((rc = launch_level(hs[q], &c[q], j, k))) return rc;
            if (lockstep) CK(hs[q], cudaEventRecord(hs[q]->ev1, hs[q]->stream));
          }
          if (!lockstep && (rc = sync_neighbours())) return rc;
        }
      for (size_t q = 0; q < n; ++q) hs[q]->cur = end_step(hs[q], &c[q]);
      // all-slab barrier + abort-word fold
      if (lockstep) continue;  // distributed semantics: aborts are reconciled by replay
      for (size_t q = 0; q < n; ++q) {
        CK(hs[q], cudaSetDevice(hs[q]->device));
        CK(hs[q], cudaEventRecord(hs[q]->ev1, hs[q]->stream));
      }
      for (size_t q = 0; q < n; ++q) {
        CK(hs[q], cudaSetDevice(hs[q]->device));
        for (size_t o = 0; o < n; ++o)
          if (o != q) CK(hs[q], cudaStreamWaitEvent(hs[q]->stream, hs[o]->ev1, 0));
        CK(hs[q], emrkc_k::launch_fold_events(hs[q]->d_event, evs.data(),
                                              static_cast<int>(n), hs[q]->stream));
      }
    }
  }
  for (size_t q = 0; q < n; ++q) {
    in_idx[q][nsteps] = hs[q]->cur;
    CK(hs[q], cudaSetDevice(hs[q]->device));
    CK(hs[q], cudaEventRecord(hs[q]->ev1, hs[q]->stream));
  }
  double ms = 0.0;
  unsigned long long ev = kNoEvent;
  std::vector<unsigned long long> slots;
  std::vector<unsigned long long> all_slots(2 * (nsteps + 1));
  for (size_t q = 0; q < n; ++q) {
    emrkc_handle* h = hs[q];
    CK(h, cudaSetDevice(h->device));
    CK(h, cudaEventSynchronize(h->ev1));
    float f = 0.0f;
    CK(h, cudaEventElapsedTime(&f, h->ev0, h->ev1));
    ms = std::max(ms, static_cast<double>(f));
    unsigned long long e = kNoEvent;
    CK(h, cudaMemcpy(&e, h->d_event, sizeof(e), cudaMemcpyDeviceToHost));
    ev = std::min(ev, e);
    slots.resize(2 * (nsteps + 1));
    CK(h, cudaMemcpy(slots.data(), h->d_slots, sizeof(unsigned long long) * slots.size(),
                     cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < slots.size(); k += 2) {
      all_slots[k] = q == 0 ? slots[k] : std::min(all_slots[k], slots[k]);
      all_slots[k + 1] = q == 0 ? slots[k + 1] : std::max(all_slots[k + 1], slots[k + 1]);
    }
  }
  if (ev == 0)
    return set_err(hs[0], EMRKC_ECUDA,
                   "distributed run: a neighbour's halo planes never arrived (10 s); "
                   "all linked slabs must run concurrently");
  Decoded d = decode_event(ev, pl);
  if (single_step && !d.none && d.guard) d = Decoded{};  // emrkc_step has no guard
  int64_t accepted = nsteps, done = nsteps;
  if (!d.none) {
    if (d.guard) {
      done = d.step + 1;
      accepted = d.step;
      for (size_t q = 0; q < n; ++q) hs[q]->cur = in_idx[q][d.step + 1];
    } else {
      done = d.step;
      accepted = d.step;
      for (size_t q = 0; q < n; ++q) hs[q]->cur = in_idx[q][d.step];
    }
  }
  if (n > 1 && !d.none) {
    // the ghost slots no longer match the (rolled back) state: the next run
    // re-exchanges from the current state.
  }
  if (res) {
    std::memset(res, 0, sizeof(*res));
    res->n_steps = nsteps;
    res->steps_done = done;
    res->aborted = d.none ? 0 : 1;
    res->abort_kind = d.none ? EMRKC_ABORT_NONE
                             : (d.guard ? EMRKC_ABORT_NORM_GUARD : EMRKC_ABORT_NONFINITE);
    res->abort_step = d.none ? -1 : step0 + d.step;
    res->abort_stage = d.guard ? 0 : d.stage;
    res->abort_inner = d.guard ? 0 : d.inner;
    res->abort_outer_stage = d.guard ? 0 : d.outer_stage;
    // track_gate_range: initial state then each accepted step (simulate.cpp:113,228)
    double lo = 1.0, hi = 0.0;
    auto fold = [&](size_t k) {
      if (all_slots[k] != kNoEvent) {
        const double v = emrkc_k::double_of(all_slots[k]);
        lo = (v < lo) ? v : lo;
      }
      if (all_slots[k + 1] != 0ull) {
        const double v = emrkc_k::double_of(all_slots[k + 1]);
        hi = (hi < v) ? v : hi;
      }
    };
    fold(2 * nsteps);
    for (int64_t r = 0; r < accepted; ++r) fold(2 * r);
    res->gate_min = lo;
    res->gate_max = hi;
    res->n_fF = done * pl.s * pl.m;
    res->n_fS = done * pl.s;
    res->n_exp = done * exp_per_step(pl.method, pl.s);
    if (!d.none && !d.guard) partial_counters(d, pl, &res->n_fF, &res->n_fS, &res->n_exp);
    // plan of the last accepted step (RunResult::steps.back(),
    // P/src/simulate.cpp:205); none when no step was accepted
    res->s = done > 0 ? pl.s : 0;
    res->m = done > 0 ? pl.m : 0;
    res->eta = done > 0 ? pl.eta : 0.0;
    res->device_ms = ms;
    if (launch_ms) {
      double tot = 0.0;
      for (int64_t i = 0; i < nsteps * pl.s * pl.m; ++i) tot += launch_ms[i];
      res->device_ms = tot;
    }
  }
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->s = pl.s;
    rep->m = pl.m;
    rep->eta = pl.eta;
    rep->ell_s = pl.ell_s;
    rep->ell_m = pl.ell_m;
    rep->n_fF = static_cast<int64_t>(pl.s) * pl.m;
    rep->n_fS = pl.s;
    rep->n_exp = exp_per_step(pl.method, pl.s);
    if (!d.none && !d.guard) {
      rep->n_fF = rep->n_fS = rep->n_exp = 0;
      partial_counters(d, pl, &rep->n_fF, &rep->n_fS, &rep->n_exp);
      rep->abort_kind = EMRKC_ABORT_NONFINITE;
      rep->abort_stage = d.stage;
      rep->abort_inner = d.inner;
      rep->abort_outer_stage = d.outer_stage;
      return set_err(hs[0], EMRKC_ENONFINITE, "rkc_iteration: non-finite value at stage %d",
                     d.stage);
    }
  }
  return EMRKC_OK;
}

}  // namespace

extern "C" {

int emrkc_estimate_rho(emrkc_handle* h, int32_t which, double t,
                       const double* v0, double rho0, emrkc_rho_result* out,
                       double* v_out) {
  if (!h || !out) return set_global(EMRKC_EINVAL, "null argument");
  if (h->partitioned)
    return set_err(h, EMRKC_EINVAL, "estimate_rho: partitioned handles use emrkc_group_estimate_rho");
  int code = 0;
  if (rhs_code(h, which, &code))
    return set_err(h, EMRKC_EINVAL, "estimate_rho: unknown rhs %d", which);
  return power_iteration({h}, code, t, v0, rho0, out, v_out);
}

namespace {
int step_impl(emrkc_handle* h, double t, double dt, double epsilon, double rho_F,
              double rho_S, emrkc_step_report* report);
}  // namespace

int emrkc_step(emrkc_handle* h, double t, double dt, double epsilon,
               int32_t variant, double rho_F, double rho_S,
               emrkc_step_report* report) {
  if (!h) return set_global(EMRKC_EINVAL, "null handle");
  if (variant_method(variant, &h->method))
    return set_err(h, EMRKC_EINVAL, "emrkc_step: unknown variant %d", variant);
  return step_impl(h, t, dt, epsilon, rho_F, rho_S, report);
}

int emrkc_exex_step(emrkc_handle* h, double t, double dt, emrkc_step_report* report) {
  if (!h) return set_global(EMRKC_EINVAL, "null handle");
  if (!(dt > 0.0)) return set_err(h, EMRKC_EINVAL, "exex_rl_step: dt must be > 0");
  h->method = kMethodExexRl;
  return step_impl(h, t, dt, 0.05, 0.0, 0.0, report);
}

namespace {
int step_impl(emrkc_handle* h, double t, double dt, double epsilon, double rho_F,
              double rho_S, emrkc_step_report* report) {
  if (h->partitioned) return set_err(h, EMRKC_EINVAL, "emrkc_step: whole-grid handles only");
  if (!(dt > 0.0)) return set_err(h, EMRKC_EINVAL, "emrkc_step: dt must be > 0");
  if (!h->has_state) return set_err(h, EMRKC_ESTATE, "no state uploaded");
  int rc = use_device(h);
  if (rc) return rc;
  if ((rc = upload_plan(h, dt, rho_F, rho_S, epsilon))) return rc;
  if ((rc = ensure_slots(h, 1))) return rc;
  const unsigned long long init[2] = {kNoEvent, 0ull};
  CK(h, cudaMemcpyAsync(h->d_event, &kNoEvent, sizeof(kNoEvent), cudaMemcpyHostToDevice,
                        h->stream));
  CK(h, cudaMemcpyAsync(h->d_slots, init, sizeof(init), cudaMemcpyHostToDevice, h->stream));
  const int in = h->cur;
  int outi = 0;
  if ((rc = enqueue_step(h, t, 0, h->d_slots, &outi))) return rc;
  unsigned long long ev = kNoEvent;
  CK(h, cudaMemcpyAsync(&ev, h->d_event, sizeof(ev), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  Decoded d = decode_event(ev, h->plan);
  if (!d.none && d.guard) d = Decoded{};  // the guard belongs to the run loop
  const Plan& pl = h->plan;
  emrkc_step_report local;
  emrkc_step_report* rep = report ? report : &local;
  std::memset(rep, 0, sizeof(*rep));
  rep->s = pl.s;
  rep->m = pl.m;
  rep->eta = pl.eta;
  rep->ell_s = pl.ell_s;
  rep->ell_m = pl.ell_m;
  rep->n_fF = static_cast<int64_t>(pl.s) * pl.m;
  rep->n_fS = pl.s;
  rep->n_exp = exp_per_step(pl.method, pl.s);
  if (d.none) {
    h->cur = outi;
    return EMRKC_OK;
  }
  h->cur = in;  // NumericalAbort: y is not assigned (P/src/simulate.cpp:215-220)
  rep->n_fF = rep->n_fS = rep->n_exp = 0;
  partial_counters(d, pl, &rep->n_fF, &rep->n_fS, &rep->n_exp);
  rep->abort_kind = EMRKC_ABORT_NONFINITE;
  rep->abort_stage = d.stage;
  rep->abort_inner = d.inner;
  rep->abort_outer_stage = d.outer_stage;
  return set_err(h, EMRKC_ENONFINITE, "rkc_iteration: non-finite value at stage %d", d.stage);
}
}  // namespace

namespace {
// emrkc_step_host for one-outer-stage steps (s = 1, any m, on the TMA
// kernels): the state crosses the host link in z-chunks on two copy
// streams. Stencil level k's range lags the copy-in chunks by k planes
// (plane p of level k needs level k - 1 at p + 1), so the levels of range
// c start as soon as copy-in chunk c has arrived and the last level's
// output goes back at once: host->device copies, the step and
// device->host copies overlap. The abort word is only known after
// the last range, so on a NumericalAbort y_out has already received (part
// of) the rejected step; the device state stays y_in (P/src/simulate.cpp:
// 215-220). Callers whose y_out overlaps y_in take the unpipelined path, so
// their input survives an abort as it does in the reference (which throws
// before assigning y).
constexpr int kMaxHostChunks = 64;

int host_chunks() {  // EMRKC_HOST_CHUNKS (default 8)
  static int n = 0;
  if (!n) {
    const char* e = std::getenv("EMRKC_HOST_CHUNKS");
    n = (e && *e) ? std::max(1, std::min(kMaxHostChunks, std::atoi(e))) : 8;
  }
  return n;
}

bool step_host_pipelined(emrkc_handle* h) {
  const Plan& pl = h->plan;
  return !h->partitioned && h->fast && h->pipe == 3 && pl.s == 1 && pl.method != kMethodMrkc &&
         !use_tb(h, pl) && host_chunks() > 1 &&
         h->geom.nzl >= (pl.m + 1) * host_chunks();
}

int step_host_pipe(emrkc_handle* h, double t, const double* y_in, double* y_out,
                   emrkc_step_report* report) {
  const int kHostChunks = host_chunks();
  if (!h->s_in) {
    CK(h, cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
    CK(h, cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
    h->ev_in.resize(kMaxHostChunks);
    h->ev_k.resize(kMaxHostChunks);
    for (int i = 0; i < kMaxHostChunks; ++i) {
      CK(h, cudaEventCreateWithFlags(&h->ev_in[i], cudaEventDisableTiming));
      CK(h, cudaEventCreateWithFlags(&h->ev_k[i], cudaEventDisableTiming));
    }
  }
  const int64_t nn = h->nn, plane = h->geom.plane;
  const int nz = h->geom.nzl;
  auto zc = [&](int c) { return static_cast<int>(static_cast<int64_t>(c) * nz / kHostChunks); };
  // Kernel / copy-out ranges lag the copy-in chunks: plane p of stencil
  // level k needs level k - 1 (or the input) at p + 1, so level k of chunk c
  // covers [zc(c) - k, zc(c+1) - k) and starts as soon as chunk c is in and
  // level k - 1 of chunk c is done (same stream); the output of the last
  // level goes out at once.
  const int m = h->plan.m;
  auto kr = [&](int c, int k) {
    return c == 0 ? 0 : (c == kHostChunks ? nz : zc(c) - k);
  };
  // abort word = no event (all ones), gate-range slots {min: all ones, max: 0}
  CK(h, cudaMemsetAsync(h->d_event, 0xff, sizeof(unsigned long long), h->stream));
  CK(h, cudaMemsetAsync(h->d_slots, 0xff, sizeof(unsigned long long), h->stream));
  CK(h, cudaMemsetAsync(h->d_slots + 1, 0, sizeof(unsigned long long), h->stream));
  CK(h, cudaEventRecord(h->ev0, h->stream));
  CK(h, cudaStreamWaitEvent(h->s_in, h->ev0, 0));  // previous use of the buffers is done
  const int in = h->cur;
  double* din = h->buf[in];
  const size_t pitch = sizeof(double) * nn;  // one row per SoA field
  for (int c = 0; c < kHostChunks; ++c) {
    const int64_t off = zc(c) * plane, n = (zc(c + 1) - zc(c)) * plane;
    CK(h, cudaMemcpy2DAsync(din + off, pitch, y_in + off, pitch, sizeof(double) * n, h->geom.nf,
                            cudaMemcpyHostToDevice, h->s_in));
    CK(h, cudaEventRecord(h->ev_in[c], h->s_in));
  }
  StepCtx sc;
  begin_step(h, t, 0, h->d_slots, &sc);
  const int outi = end_step(h, &sc);
  int rc = EMRKC_OK;
  for (int c = 0; c < kHostChunks && !rc; ++c) {
    CK(h, cudaStreamWaitEvent(h->stream, h->ev_in[c], 0));
    for (int k = 1; k <= m && !rc; ++k) {
      h->zr_lo = kr(c, k);
      h->zr_hi = kr(c + 1, k);
      rc = launch_level(h, &sc, 1, k);
    }
    CK(h, cudaEventRecord(h->ev_k[c], h->stream));
  }
  h->zr_lo = h->zr_hi = -1;
  if (rc) {
    // copies from the caller's y_in may still be in flight into buf[in]:
    // drain every stream before handing control (and y_in) back, and drop
    // the device state, which is partly written
    cudaStreamSynchronize(h->s_in);
    cudaStreamSynchronize(h->stream);
    cudaStreamSynchronize(h->s_out);
    h->has_state = false;
    return rc;
  }
  double* dout = h->buf[outi];
  for (int c = 0; c < kHostChunks; ++c) {
    CK(h, cudaStreamWaitEvent(h->s_out, h->ev_k[c], 0));
    const int64_t off = kr(c, m) * plane, n = (kr(c + 1, m) - kr(c, m)) * plane;
    CK(h, cudaMemcpy2DAsync(y_out + off, pitch, dout + off, pitch, sizeof(double) * n, h->geom.nf,
                            cudaMemcpyDeviceToHost, h->s_out));
  }
  if (!h->h_event) CK(h, cudaHostAlloc(&h->h_event, sizeof(unsigned long long), 0));
  CK(h, cudaMemcpyAsync(h->h_event, h->d_event, sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  CK(h, cudaStreamSynchronize(h->s_out));
  const unsigned long long ev = *h->h_event;
  h->has_state = true;
  Decoded d = decode_event(ev, h->plan);
  if (!d.none && d.guard) d = Decoded{};  // the guard belongs to the run loop
  const Plan& pl = h->plan;
  emrkc_step_report local;
  emrkc_step_report* rep = report ? report : &local;
  std::memset(rep, 0, sizeof(*rep));
  rep->s = pl.s;
  rep->m = pl.m;
  rep->eta = pl.eta;
  rep->ell_s = pl.ell_s;
  rep->ell_m = pl.ell_m;
  rep->n_fF = static_cast<int64_t>(pl.s) * pl.m;
  rep->n_fS = pl.s;
  rep->n_exp = exp_per_step(pl.method, pl.s);
  if (d.none) {
    h->cur = outi;
    return EMRKC_OK;
  }
  h->cur = in;  // NumericalAbort: y is not assigned (P/src/simulate.cpp:215-220)
  rep->n_fF = rep->n_fS = rep->n_exp = 0;
  partial_counters(d, pl, &rep->n_fF, &rep->n_fS, &rep->n_exp);
  rep->abort_kind = EMRKC_ABORT_NONFINITE;
  rep->abort_stage = d.stage;
  rep->abort_inner = d.inner;
  rep->abort_outer_stage = d.outer_stage;
  return set_err(h, EMRKC_ENONFINITE, "rkc_iteration: non-finite value at stage %d", d.stage);
}
}  // namespace

int emrkc_step_host(emrkc_handle* h, double t, const double* y_in,
                    double* y_out, int64_t len, double dt, double epsilon,
                    int32_t variant, double rho_F, double rho_S,
                    emrkc_step_report* report) {
  if (!h || !y_in || !y_out) return set_global(EMRKC_EINVAL, "null argument");
  if (!h->partitioned && len == h->len && (dt > 0.0) && !variant_method(variant, &h->method)) {
    int rc = use_device(h);
    if (rc) return rc;
    if ((rc = ensure_buffers(h, std::max(2, h->nbuf)))) return rc;
    if ((rc = upload_plan(h, dt, rho_F, rho_S, epsilon))) return rc;
    if ((rc = ensure_slots(h, 1))) return rc;
    const bool overlap = y_out < y_in + len && y_in < y_out + len;
    if (!overlap && step_host_pipelined(h)) return step_host_pipe(h, t, y_in, y_out, report);
  }
  int rc = emrkc_set_state(h, y_in, len);
  if (rc) return rc;
  rc = emrkc_step(h, t, dt, epsilon, variant, rho_F, rho_S, report);
  if (rc) return rc;
  return emrkc_get_state(h, y_out, len);
}

int emrkc_run(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt,
              double epsilon, int32_t variant, double rho_F, double rho_S,
              emrkc_run_result* res) {
  if (!h || !res) return set_global(EMRKC_EINVAL, "null argument");
  if (h->partitioned) return set_err(h, EMRKC_EINVAL, "emrkc_run: whole-grid handles only");
  if (variant_method(variant, &h->method))
    return set_err(h, EMRKC_EINVAL, "emrkc_run: unknown variant %d", variant);
  if (nsteps < 0) return set_err(h, EMRKC_EINVAL, "emrkc_run: nsteps must be >= 0");
  return run_slabs({h}, step0, nsteps, dt, epsilon, rho_F, rho_S, res, false, nullptr);
}

int emrkc_exex_run(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt,
                   emrkc_run_result* res) {
  if (!h || !res) return set_global(EMRKC_EINVAL, "null argument");
  if (h->partitioned) return set_err(h, EMRKC_EINVAL, "emrkc_exex_run: whole-grid handles only");
  if (!(dt > 0.0)) return set_err(h, EMRKC_EINVAL, "exex_rl_step: dt must be > 0");
  if (nsteps < 0) return set_err(h, EMRKC_EINVAL, "emrkc_exex_run: nsteps must be >= 0");
  h->method = kMethodExexRl;
  return run_slabs({h}, step0, nsteps, dt, 0.05, 0.0, 0.0, res, false, nullptr);
}

int emrkc_set_stiff_gates(emrkc_handle* h, int32_t mask) {
  if (!h) return set_global(EMRKC_EINVAL, "null handle");
  if (mask < 0 || mask > 7) return set_err(h, EMRKC_EINVAL, "stiff gate mask must be 0..7");
  h->stiff = mask;
  h->plan_uploaded = false;
  return EMRKC_OK;
}

int emrkc_identify_stiff_gates(int32_t model, const double* V, int64_t n, int32_t* order) {
  if (model != EMRKC_MODEL_HH) return set_global(EMRKC_EINVAL, "unknown ionic model %d", model);
  if (!V || !order) return set_global(EMRKC_EINVAL, "null argument");
  if (n < 1) return set_global(EMRKC_EINVAL, "identify_stiff_gates: empty trajectory");
  double mr[3] = {0.0, 0.0, 0.0};  // max alpha + beta per gate (P/src/ionic.cpp:133-140)
  for (int64_t i = 0; i < n; ++i) {
    double a[3], b[3];
    hh_rates(V[i], a, b);
    for (int g = 0; g < 3; ++g) mr[g] = std::max(mr[g], a[g] + b[g]);
  }
  int o[3] = {0, 1, 2};
  std::stable_sort(o, o + 3, [&](int x, int y) { return mr[x] > mr[y]; });
  for (int g = 0; g < 3; ++g) order[g] = o[g];
  return EMRKC_OK;
}

namespace {
int ensure_mrkc(emrkc_handle* h) {
  for (auto& u : h->mr_u)
    if (!u) CK(h, cudaMalloc(&u, sizeof(double) * h->len));
  if (!h->mr_fs) CK(h, cudaMalloc(&h->mr_fs, sizeof(double) * h->len));
  return EMRKC_OK;
}
}  // namespace

int emrkc_mrkc_step(emrkc_handle* h, double t, double dt, double epsilon, double rho_F,
                    double rho_S, emrkc_step_report* report) {
  if (!h) return set_global(EMRKC_EINVAL, "null handle");
  if (!(dt > 0.0)) return set_err(h, EMRKC_EINVAL, "mrkc_step: dt must be > 0");
  int rc = use_device(h);
  if (rc) return rc;
  if ((rc = ensure_mrkc(h))) return rc;
  h->method = kMethodMrkc;
  return step_impl(h, t, dt, epsilon, rho_F, rho_S, report);
}

int emrkc_mrkc_run(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt, double epsilon,
                   double rho_F, double rho_S, emrkc_run_result* res) {
  if (!h || !res) return set_global(EMRKC_EINVAL, "null argument");
  if (h->partitioned) return set_err(h, EMRKC_EINVAL, "emrkc_mrkc_run: whole-grid handles only");
  if (nsteps < 0) return set_err(h, EMRKC_EINVAL, "emrkc_mrkc_run: nsteps must be >= 0");
  int rc = use_device(h);
  if (rc) return rc;
  if ((rc = ensure_mrkc(h))) return rc;
  h->method = kMethodMrkc;
  return run_slabs({h}, step0, nsteps, dt, epsilon, rho_F, rho_S, res, false, nullptr);
}

namespace {
// One imex_rl_step (P/src/baselines.cpp:132-190) of buf[cur] into the other
// buffer. Returns 0 with *ok = 0 when CG did not converge (NumericalAbort).
int imex_step_dev(emrkc_handle* h, double t, double dt, double rel_tol, int64_t max_iters,
                  int jacobi, int* ok, int64_t* iters, int* guard) {
  const int64_t nn = h->nn;
  const int nb = emrkc_k::power_blocks();
  if (!h->cg_v) CK(h, cudaMalloc(&h->cg_v, sizeof(double) * 6 * nn));
  if (!h->cg_part) CK(h, cudaMalloc(&h->cg_part, sizeof(double) * 3 * nb));
  if (!h->cg_s) CK(h, cudaMalloc(&h->cg_s, sizeof(emrkc_k::CgScalars)));
  if (!h->cg_h) CK(h, cudaHostAlloc(&h->cg_h, sizeof(emrkc_k::CgScalars), 0));
  if (!h->guard_d) CK(h, cudaMalloc(&h->guard_d, sizeof(int)));
  double* b = h->cg_v;
  double* x = b + nn;
  double* r = x + nn;
  double* z = r + nn;
  double* pp = z + nn;
  double* q = pp + nn;
  double* part = h->cg_part;        // 2 nb
  double* part_b = h->cg_part + 2 * nb;  // nb
  const int in = h->cur, out = 1 - (h->cur & 1);
  double* y = h->buf[in];
  double* yo = h->buf[out];
  // diag(I - dt D): constant for the reflection stencil (:171-177)
  const double diag = jacobi ? 1.0 - dt * emrkc_k::diffusion_diag(h->geom) : 0.0;
  const long long max_it = max_iters > 0
                               ? max_iters
                               : static_cast<long long>(10.0 * std::sqrt(static_cast<double>(nn))) + 1;
  CK(h, emrkc_k::launch_imex_prep(h->geom, y, dt, stim_rate_at(&h->p, t), yo, b, x, part_b, nb,
                                  h->stream));
  CK(h, emrkc_k::launch_cg_init(h->geom, dt, diag, b, x, r, z, pp, part, nb, h->cg_s, rel_tol,
                                max_it, part_b, h->stream));
  constexpr int kBatch = 8;  // iterations between host checks of the loop test
  for (long long done_it = 0;; done_it += kBatch) {
    for (int i = 0; i < kBatch; ++i)
      CK(h, emrkc_k::launch_cg_iter(h->geom, dt, diag, x, r, z, pp, q, part, nb, h->cg_s,
                                    h->stream));
    CK(h, cudaMemcpyAsync(h->cg_h, h->cg_s, sizeof(emrkc_k::CgScalars),
                          cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    if (h->cg_h->done || done_it > max_it + kBatch) break;
  }
  CK(h, emrkc_k::launch_cg_finish(h->geom, x, yo, h->cg_s, h->stream));
  CK(h, cudaMemsetAsync(h->guard_d, 0, sizeof(int), h->stream));
  CK(h, emrkc_k::launch_v_guard(nn, yo, h->guard_d, h->stream));
  int g = 0;
  CK(h, cudaMemcpyAsync(&g, h->guard_d, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  *ok = h->cg_h->converged && h->cg_h->done;
  *iters = h->cg_h->it;
  *guard = g;
  return EMRKC_OK;
}
}  // namespace

int emrkc_imex_step(emrkc_handle* h, double t, double dt, double rel_tol, int64_t max_iters,
                    int32_t jacobi, emrkc_step_report* report, int64_t* cg_iters) {
  if (!h) return set_global(EMRKC_EINVAL, "null handle");
  if (h->partitioned) return set_err(h, EMRKC_EINVAL, "imex_rl_step: whole-grid handles only");
  if (h->geom.naux > 0) return set_err(h, EMRKC_EINVAL, "imex_rl_step: HH only");
  if (!(dt > 0.0)) return set_err(h, EMRKC_EINVAL, "imex_rl_step: dt must be > 0");
  if (!h->has_state) return set_err(h, EMRKC_ESTATE, "no state uploaded");
  int rc = use_device(h);
  if (rc) return rc;
  if ((rc = ensure_buffers(h, std::max(2, h->nbuf)))) return rc;
  int ok = 0, guard = 0;
  int64_t it = 0;
  if ((rc = imex_step_dev(h, t, dt, rel_tol, max_iters, jacobi, &ok, &it, &guard))) return rc;
  emrkc_step_report local;
  emrkc_step_report* rep = report ? report : &local;
  std::memset(rep, 0, sizeof(*rep));
  rep->s = rep->m = 1;
  rep->eta = dt;
  rep->n_fF = it + 2;  // CG applies (iterations + 1) + the diagonal probe
  rep->n_fS = 1;
  rep->n_exp = 1;
  if (cg_iters) *cg_iters = it;
  if (!ok) {
    rep->abort_kind = EMRKC_ABORT_NONFINITE;
    rep->abort_stage = -1;
    return set_err(h, EMRKC_ENONFINITE, "imex_rl_step: CG did not converge");
  }
  h->cur = 1 - (h->cur & 1);
  return EMRKC_OK;
}

int emrkc_imex_run(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt, double rel_tol,
                   int64_t max_iters, int32_t jacobi, emrkc_run_result* res,
                   int64_t* cg_iters_total) {
  if (!h || !res) return set_global(EMRKC_EINVAL, "null argument");
  if (h->partitioned) return set_err(h, EMRKC_EINVAL, "imex_rl_step: whole-grid handles only");
  if (h->geom.naux > 0) return set_err(h, EMRKC_EINVAL, "imex_rl_step: HH only");
  if (!(dt > 0.0)) return set_err(h, EMRKC_EINVAL, "imex_rl_step: dt must be > 0");
  if (nsteps < 0) return set_err(h, EMRKC_EINVAL, "emrkc_imex_run: nsteps must be >= 0");
  if (!h->has_state) return set_err(h, EMRKC_ESTATE, "no state uploaded");
  int rc = use_device(h);
  if (rc) return rc;
  if ((rc = ensure_buffers(h, std::max(2, h->nbuf)))) return rc;
  if ((rc = ensure_slots(h, 1))) return rc;
  std::memset(res, 0, sizeof(*res));
  res->n_steps = nsteps;
  res->abort_step = -1;
  res->s = res->m = 1;
  res->eta = dt;
  // gate range of the initial state and of every accepted step (simulate.cpp:113,228)
  const unsigned long long init[2] = {kNoEvent, 0ull};
  CK(h, cudaMemcpyAsync(h->d_slots, init, sizeof(init), cudaMemcpyHostToDevice, h->stream));
  CK(h, emrkc_k::launch_gate_range(h->geom, h->buf[h->cur], h->d_slots, h->stream));
  int64_t iters_total = 0;
  CK(h, cudaEventRecord(h->ev0, h->stream));
  for (int64_t s = 0; s < nsteps; ++s) {
    const int64_t step = step0 + s;
    const double t = static_cast<double>(step) * dt;  // simulate.cpp:177
    int ok = 0, guard = 0;
    int64_t it = 0;
    if ((rc = imex_step_dev(h, t, dt, rel_tol, max_iters, jacobi, &ok, &it, &guard))) return rc;
    res->n_fF += it + 2;
    res->n_fS += 1;
    res->n_exp += 1;
    iters_total += it;
    if (!ok) {  // NumericalAbort: y is not assigned
      res->aborted = 1;
      res->abort_kind = EMRKC_ABORT_NONFINITE;
      res->abort_step = step;
      res->abort_stage = -1;
      break;
    }
    h->cur = 1 - (h->cur & 1);
    ++res->steps_done;
    if (guard) {
      res->aborted = 1;
      res->abort_kind = EMRKC_ABORT_NORM_GUARD;
      res->abort_step = step;
      break;
    }
    CK(h, emrkc_k::launch_gate_range(h->geom, h->buf[h->cur], h->d_slots, h->stream));
  }
  CK(h, cudaEventRecord(h->ev1, h->stream));
  unsigned long long sl[2];
  CK(h, cudaMemcpyAsync(sl, h->d_slots, sizeof(sl), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  // track_gate_range from gate_min = 1, gate_max = 0 (simulate.cpp:111-113)
  res->gate_min = 1.0;
  res->gate_max = 0.0;
  if (sl[0] != kNoEvent) res->gate_min = std::min(1.0, emrkc_k::double_of(sl[0]));
  if (sl[1] != 0ull) res->gate_max = std::max(0.0, emrkc_k::double_of(sl[1]));
  float ms = 0.0f;
  CK(h, cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  res->device_ms = ms;
  if (cg_iters_total) *cg_iters_total = iters_total;
  return EMRKC_OK;
}

int emrkc_run_timed(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt,
                    double epsilon, int32_t variant, double rho_F,
                    double rho_S, int64_t flush_bytes, double* launch_ms,
                    int64_t launch_ms_len, emrkc_run_result* res) {
  if (!h || !res || !launch_ms) return set_global(EMRKC_EINVAL, "null argument");
  if (h->partitioned && !dist_linked(h) && !(h->z_begin == 0 && h->z_end == h->p.n[h->p.dim - 1]))
    return set_err(h, EMRKC_EINVAL, "emrkc_run_timed: whole-grid or distributed handles only");
  if (variant_method(variant, &h->method))
    return set_err(h, EMRKC_EINVAL, "emrkc_run: unknown variant %d", variant);
  if (nsteps < 0 || flush_bytes < 0) return set_err(h, EMRKC_EINVAL, "emrkc_run_timed: bad sizes");
  return run_slabs({h}, step0, nsteps, dt, epsilon, rho_F, rho_S, res, false, nullptr,
                   flush_bytes, launch_ms, launch_ms_len);
}

// ---- groups ---------------------------------------------------------------

int emrkc_group_create(emrkc_handle* const* hs, int32_t n, emrkc_group** out) {
  if (!hs || n < 1 || !out) return set_global(EMRKC_EINVAL, "group: bad arguments");
  *out = nullptr;
  const emrkc_problem& p0 = hs[0]->p;
  int64_t z = 0;
  for (int r = 0; r < n; ++r) {
    emrkc_handle* h = hs[r];
    if (!h) return set_global(EMRKC_EINVAL, "group: null handle");
    if (std::memcmp(&h->p, &p0, sizeof(p0)) != 0)
      return set_global(EMRKC_EINVAL, "group: handles describe different problems");
    if (h->z_begin != z)
      return set_global(EMRKC_EINVAL, "group: slabs must be consecutive and ordered");
    z = h->z_end;
    if (h->nbr[0] || h->nbr[1])
      return set_global(EMRKC_EINVAL, "group: handle already linked");
  }
  if (z != p0.n[p0.dim - 1])
    return set_global(EMRKC_EINVAL, "group: slabs do not cover the grid");
  int64_t min_depth = z;
  for (int r = 0; r < n; ++r) min_depth = std::min(min_depth, hs[r]->z_end - hs[r]->z_begin);
  for (int r = 0; r < n; ++r) {
    hs[r]->nbr[0] = r > 0 ? hs[r - 1] : nullptr;
    hs[r]->nbr[1] = r + 1 < n ? hs[r + 1] : nullptr;
    hs[r]->level = 0;
    hs[r]->kstage = 0;
    hs[r]->min_depth = min_depth;
    // peer access for stores into neighbours on other devices
    for (int o = 0; o < n; ++o) {
      if (hs[o]->device == hs[r]->device) continue;
      cudaSetDevice(hs[r]->device);
      const cudaError_t e = cudaDeviceEnablePeerAccess(hs[o]->device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return set_global(EMRKC_ECUDA, "group: peer access %d->%d: %s", hs[r]->device,
                          hs[o]->device, cudaGetErrorString(e));
      cudaGetLastError();
    }
  }
  auto* g = new emrkc_group();
  g->hs.assign(hs, hs + n);
  *out = g;
  return EMRKC_OK;
}

void emrkc_group_destroy(emrkc_group* g) {
  if (!g) return;
  for (auto* h : g->hs) {
    h->nbr[0] = h->nbr[1] = nullptr;
  }
  delete g;
}

int emrkc_group_estimate_rho(emrkc_group* g, int32_t which, double t,
                             emrkc_rho_result* out) {
  if (!g || !out) return set_global(EMRKC_EINVAL, "null argument");
  if (which != EMRKC_RHS_F && which != EMRKC_RHS_S)
    return set_global(EMRKC_EINVAL, "estimate_rho: which must be F or S");
  return power_iteration(g->hs, which, t, nullptr, 0.0, out, nullptr);
}

int emrkc_group_run(emrkc_group* g, int64_t step0, int64_t nsteps, double dt,
                    double epsilon, int32_t variant, double rho_F,
                    double rho_S, emrkc_run_result* res) {
  if (!g || !res) return set_global(EMRKC_EINVAL, "null argument");
  int method = 0;
  if (variant_method(variant, &method))
    return set_global(EMRKC_EINVAL, "emrkc_run: unknown variant %d", variant);
  for (auto* h : g->hs) h->method = method;
  return run_slabs(g->hs, step0, nsteps, dt, epsilon, rho_F, rho_S, res, false, nullptr);
}

// ---- multi-process ----------------------------------------------------------

namespace {
struct IpcBlob {
  char magic[8];
  int32_t version;
  int32_t device;
  int64_t plane;
  int64_t z_begin, z_end;
  int64_t arena_bytes;
  cudaIpcMemHandle_t mem;
};
constexpr char kBlobMagic[8] = {'E', 'M', 'R', 'K', 'C', 'I', 'P', 'C'};

// Points side s of h at a neighbour arena (ghost[1-s][*] and cnt[1-s]).
void link_peer(emrkc_handle* h, int s, void* arena, bool ipc) {
  const size_t pl = static_cast<size_t>(h->geom.plane);
  double* base = static_cast<double*>(arena);
  const int o = 1 - s;
  h->peer[s].linked = true;
  h->peer[s].ipc = ipc;
  h->peer[s].arena = arena;
  h->peer[s].ghost[0] = base + (2 * o + 0) * pl;
  h->peer[s].ghost[1] = base + (2 * o + 1) * pl;
  for (int par = 0; par < 2; ++par)
    h->peer[s].dghost[par] = h->geom.dim == 3 ? dghost_at(base, pl, o, par) : nullptr;
  h->peer[s].cnt =
      reinterpret_cast<unsigned long long*>(base + arena_planes(h->geom.dim) * pl) + o;
}
}  // namespace

int64_t emrkc_ipc_blob_size(void) { return static_cast<int64_t>(sizeof(IpcBlob)); }

int emrkc_ipc_export(emrkc_handle* h, void* blob, int64_t len) {
  if (!h || !blob || len < static_cast<int64_t>(sizeof(IpcBlob)))
    return set_global(EMRKC_EINVAL, "ipc_export: bad arguments");
  if (!h->partitioned || !h->arena)
    return set_err(h, EMRKC_EINVAL, "ipc_export: handle is not a partitioned slab");
  int rc = use_device(h);
  if (rc) return rc;
  IpcBlob b{};
  std::memcpy(b.magic, kBlobMagic, 8);
  b.version = EMRKC_ABI_VERSION;
  b.device = h->device;
  b.plane = h->geom.plane;
  b.z_begin = h->z_begin;
  b.z_end = h->z_end;
  b.arena_bytes = static_cast<int64_t>(h->arena_bytes);
  CK(h, cudaIpcGetMemHandle(&b.mem, h->arena));
  std::memcpy(blob, &b, sizeof(b));
  return EMRKC_OK;
}

int emrkc_ipc_import(emrkc_handle* h, int32_t side, const void* blob, int64_t len) {
  if (!h || !blob || len < static_cast<int64_t>(sizeof(IpcBlob)) || (side != 0 && side != 1))
    return set_global(EMRKC_EINVAL, "ipc_import: bad arguments");
  IpcBlob b;
  std::memcpy(&b, blob, sizeof(b));
  if (std::memcmp(b.magic, kBlobMagic, 8) != 0 || b.version != EMRKC_ABI_VERSION)
    return set_err(h, EMRKC_EINVAL, "ipc_import: not an emrkc blob");
  if (b.plane != h->geom.plane)
    return set_err(h, EMRKC_EINVAL, "ipc_import: plane size mismatch");
  if ((side == 0 && b.z_end != h->z_begin) || (side == 1 && b.z_begin != h->z_end))
    return set_err(h, EMRKC_EINVAL, "ipc_import: blob is not the %s neighbour",
                   side == 0 ? "lower" : "upper");
  int rc = use_device(h);
  if (rc) return rc;
  void* ptr = nullptr;
  CK(h, cudaIpcOpenMemHandle(&ptr, b.mem, cudaIpcMemLazyEnablePeerAccess));
  link_peer(h, side, ptr, true);
  return EMRKC_OK;
}

int emrkc_dist_run(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt,
                   double epsilon, int32_t variant, double rho_F,
                   double rho_S, emrkc_run_result* res) {
  if (!h || !res) return set_global(EMRKC_EINVAL, "null argument");
  if (variant_method(variant, &h->method))
    return set_err(h, EMRKC_EINVAL, "emrkc_run: unknown variant %d", variant);
  if (!h->partitioned) return set_err(h, EMRKC_EINVAL, "dist_run: handle is not a slab");
  return run_slabs({h}, step0, nsteps, dt, epsilon, rho_F, rho_S, res, false, nullptr);
}

int emrkc_dist_replay(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt,
                      double epsilon, int32_t variant, double rho_F, double rho_S,
                      emrkc_run_result* res) {
  if (!h || !res) return set_global(EMRKC_EINVAL, "null argument");
  if (!h->ckpt) return set_err(h, EMRKC_ESTATE, "dist_replay: no dist_run checkpoint");
  int rc = use_device(h);
  if (rc) return rc;
  CK(h, cudaMemcpyAsync(h->buf[h->cur], h->ckpt, sizeof(double) * h->len,
                        cudaMemcpyDeviceToDevice, h->stream));
  return emrkc_dist_run(h, step0, nsteps, dt, epsilon, variant, rho_F, rho_S, res);
}

int emrkc_set_slab_min_depth(emrkc_handle* h, int64_t min_planes) {
  if (!h) return set_global(EMRKC_EINVAL, "null handle");
  if (!h->partitioned) return set_err(h, EMRKC_EINVAL, "set_slab_min_depth: not a slab");
  if (min_planes < 0 || min_planes > h->z_end - h->z_begin)
    return set_err(h, EMRKC_EINVAL, "set_slab_min_depth: %lld exceeds this slab's depth",
                   (long long)min_planes);
  h->min_depth = min_planes;
  return EMRKC_OK;
}

int emrkc_set_level_hook(emrkc_handle* h, emrkc_level_hook hook, void* ctx) {
  if (!h) return set_global(EMRKC_EINVAL, "null handle");
  h->level_hook = hook;
  h->level_ctx = ctx;
  return EMRKC_OK;
}

int emrkc_dist_link_local(emrkc_handle* lower, emrkc_handle* upper) {
  if (!lower || !upper) return set_global(EMRKC_EINVAL, "null handle");
  if (lower->z_end != upper->z_begin || lower->geom.plane != upper->geom.plane ||
      !lower->arena || !upper->arena)
    return set_global(EMRKC_EINVAL, "dist_link_local: slabs are not adjacent");
  if (lower->device != upper->device) {
    cudaSetDevice(lower->device);
    cudaError_t e = cudaDeviceEnablePeerAccess(upper->device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
      return set_global(EMRKC_ECUDA, "peer access: %s", cudaGetErrorString(e));
    cudaSetDevice(upper->device);
    e = cudaDeviceEnablePeerAccess(lower->device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
      return set_global(EMRKC_ECUDA, "peer access: %s", cudaGetErrorString(e));
    cudaGetLastError();
  }
  link_peer(lower, 1, upper->arena, false);
  link_peer(upper, 0, lower->arena, false);
  return EMRKC_OK;
}

int emrkc_dist_lockstep_run(emrkc_handle* const* hs, int32_t n, int32_t replay,
                            int64_t step0, int64_t nsteps, double dt, double epsilon,
                            int32_t variant, double rho_F, double rho_S,
                            emrkc_run_result* res) {
  if (!hs || n < 1 || !res) return set_global(EMRKC_EINVAL, "bad arguments");
  int method = 0;
  if (variant_method(variant, &method))
    return set_global(EMRKC_EINVAL, "emrkc_run: unknown variant %d", variant);
  std::vector<emrkc_handle*> v(hs, hs + n);
  int64_t min_depth = v[0]->z_end - v[0]->z_begin;
  for (auto* h : v) min_depth = std::min(min_depth, h->z_end - h->z_begin);
  for (auto* h : v) {
    h->method = method;
    h->min_depth = min_depth;
  }
  for (auto* h : v) {
    if (!dist_linked(h)) return set_global(EMRKC_ESTATE, "dist_lockstep_run: handles not linked");
    if (replay) {
      if (!h->ckpt) return set_err(h, EMRKC_ESTATE, "dist replay: no checkpoint");
      cudaSetDevice(h->device);
      CK(h, cudaMemcpy(h->buf[h->cur], h->ckpt, sizeof(double) * h->len,
                       cudaMemcpyDeviceToDevice));
    }
  }
  return run_slabs(v, step0, nsteps, dt, epsilon, rho_F, rho_S, res, false, nullptr, 0,
                   nullptr, 0, /*lockstep=*/true);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// SplitRhs of a handle's operator for the generic integrator layer
// (emrkc_generic.cu): device callbacks on the caller's stream.
// ---------------------------------------------------------------------------
namespace {
int bound_rhs(emrkc_handle* h, int which, double t, const double* y, double* out, int64_t len,
              void* stream) {
  if (!h || len != h->len || h->partitioned) return 1;
  int code = 0;
  if (rhs_code(h, which, &code) || use_device(h)) return 1;
  return emrkc_k::launch_rhs(h->geom, Halo{}, code, y, stim_rate_at(&h->p, t), out,
                             static_cast<cudaStream_t>(stream)) != cudaSuccess;
}
int bound_fF(void* ctx, double t, const double* y, double* out, int64_t len, void* stream) {
  return bound_rhs(static_cast<emrkc_handle*>(ctx), EMRKC_RHS_F, t, y, out, len, stream);
}
int bound_fS(void* ctx, double t, const double* y, double* out, int64_t len, void* stream) {
  return bound_rhs(static_cast<emrkc_handle*>(ctx), EMRKC_RHS_S, t, y, out, len, stream);
}
int bound_exp(void* ctx, const double* y, double* lam, double* yinf, int64_t len, void* stream) {
  auto* h = static_cast<emrkc_handle*>(ctx);
  if (!h || len != h->len || h->partitioned || use_device(h)) return 1;
  return emrkc_k::launch_exp_part(h->geom, y, lam, yinf, static_cast<cudaStream_t>(stream)) !=
         cudaSuccess;
}
}  // namespace

int emrkc_bind_split_rhs(emrkc_handle* h, emrkc_split_rhs* out) {
  if (!h || !out) return set_global(EMRKC_EINVAL, "null argument");
  if (h->partitioned) return set_err(h, EMRKC_EINVAL, "bind_split_rhs: whole-grid handles only");
  *out = emrkc_split_rhs{};
  out->f_F = bound_fF;
  out->f_F_ctx = h;
  out->f_S = bound_fS;
  out->f_S_ctx = h;
  out->exp_part = bound_exp;
  out->exp_ctx = h;
  return EMRKC_OK;
}

int emrkc_model_rates(int32_t model, double V, double* alpha, double* beta) {
  if (model != EMRKC_MODEL_HH) return set_global(EMRKC_EINVAL, "unknown ionic model %d", model);
  if (!alpha || !beta) return set_global(EMRKC_EINVAL, "null argument");
  hh_rates(V, alpha, beta);
  return EMRKC_OK;
}

int emrkc_model_ionic_current(int32_t model, double V, const double* z_E, double* current) {
  if (model != EMRKC_MODEL_HH) return set_global(EMRKC_EINVAL, "unknown ionic model %d", model);
  if (!z_E || !current) return set_global(EMRKC_EINVAL, "null argument");
  *current = hh_current(V, z_E);
  return EMRKC_OK;
}

int32_t emrkc_node_kernel(emrkc_handle* h) {
  if (!h) return 0;
  return use_pair(h) && emrkc_k::pair_zc(h->geom, true, h->pair == 2) > 0 ? 1 : 0;
}

int32_t emrkc_fused_active(emrkc_handle* h) {
  if (!h || !h->plan_uploaded) return 0;
  if (use_fused(h, h->plan)) return 1;
  if (use_zpipe(h, h->plan)) return 2;
  return use_xstep(h, h->plan, 2) ? 3 : 0;
}

// ---------------------------------------------------------------------------
// estimate_spectral_radius over z-slabs held by separate processes
// (P/src/spectral.cpp:26-71), one primitive at a time; the host loop
// (paper_2401_01745_b200/dist.py slab_rho) moves the V ghost planes between
// ranks and chains the norms across ranks in the reference's serial order.
// ---------------------------------------------------------------------------
int emrkc_slab_power_begin(emrkc_handle* h, int32_t which, const double* v0_slab) {
  if (!h) return set_global(EMRKC_EINVAL, "null handle");
  if (!h->has_state) return set_err(h, EMRKC_ESTATE, "no state uploaded");
  int code = 0;
  if (rhs_code(h, which, &code))
    return set_err(h, EMRKC_EINVAL, "estimate_rho: unknown rhs %d", which);
  int rc = use_device(h);
  if (rc) return rc;
  for (int k = 0; k < 2; ++k)
    if (!h->sp_v[k]) CK(h, cudaMalloc(&h->sp_v[k], sizeof(double) * h->len));
  if (!h->sp_fy) CK(h, cudaMalloc(&h->sp_fy, sizeof(double) * h->len));
  std::vector<double> local;
  if (v0_slab) {
    local.assign(v0_slab, v0_slab + h->len);
  } else {  // this slab's part of the reference's seeded direction over the global state
    std::vector<double> v0(static_cast<size_t>(h->geom.nf) * nodes_of(&h->p));
    seeded_direction(v0);
    scatter_slab(h, v0, nodes_of(&h->p), local);
  }
  CK(h, cudaMemcpy(h->sp_v[0], local.data(), sizeof(double) * h->len, cudaMemcpyHostToDevice));
  h->sp_code = code;
  h->sp_a = 0;
  return EMRKC_OK;
}

int emrkc_slab_power_plane(emrkc_handle* h, int32_t field, int32_t side, double* dst) {
  if (!h || !dst) return set_global(EMRKC_EINVAL, "null argument");
  if (h->sp_code < 0) return set_err(h, EMRKC_ESTATE, "slab power iteration not begun");
  if (field < 0 || field > 1 || side < 0 || side > 1)
    return set_err(h, EMRKC_EINVAL, "slab_power_plane: field / side must be 0 or 1");
  int rc = use_device(h);
  if (rc) return rc;
  const double* x = field == 0 ? h->sp_v[h->sp_a] : h->buf[h->cur];
  const int64_t pl = h->geom.plane;
  CK(h, cudaMemcpyAsync(dst, x + (side ? h->nn - pl : 0), sizeof(double) * pl,
                        cudaMemcpyDeviceToDevice, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return EMRKC_OK;
}

int emrkc_slab_power_sumsq(emrkc_handle* h, int32_t field, int32_t block, double acc_in,
                           double* acc_out) {
  if (!h || !acc_out) return set_global(EMRKC_EINVAL, "null argument");
  if (h->sp_code < 0) return set_err(h, EMRKC_ESTATE, "slab power iteration not begun");
  if (field < 0 || field > 1 || block < 0 || block >= h->geom.nf)
    return set_err(h, EMRKC_EINVAL, "slab_power_sumsq: field 0/1, block 0..fields-1");
  int rc = use_device(h);
  if (rc) return rc;
  const double* x = (field == 0 ? h->sp_v[h->sp_a] : h->buf[h->cur]) + block * h->nn;
  CK(h, emrkc_k::launch_sumsq_serial(x, h->nn, acc_in, h->d_red, h->stream));
  CK(h, cudaMemcpyAsync(acc_out, h->d_red, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return EMRKC_OK;
}

int emrkc_slab_power_fy(emrkc_handle* h, double t, const double* gy_lo, const double* gy_hi) {
  if (!h) return set_global(EMRKC_EINVAL, "null handle");
  if (h->sp_code < 0) return set_err(h, EMRKC_ESTATE, "slab power iteration not begun");
  int rc = use_device(h);
  if (rc) return rc;
  Halo hh{};
  hh.lo = gy_lo;
  hh.hi = gy_hi;
  CK(h, emrkc_k::launch_rhs(h->geom, hh, h->sp_code, h->buf[h->cur], stim_rate_at(&h->p, t),
                            h->sp_fy, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return EMRKC_OK;
}

int emrkc_slab_power_step(emrkc_handle* h, double t, double q, const double* gy_lo,
                          const double* gy_hi, const double* gv_lo, const double* gv_hi) {
  if (!h) return set_global(EMRKC_EINVAL, "null handle");
  if (h->sp_code < 0) return set_err(h, EMRKC_ESTATE, "slab power iteration not begun");
  if ((gy_lo == nullptr) != (gv_lo == nullptr) || (gy_hi == nullptr) != (gv_hi == nullptr))
    return set_err(h, EMRKC_EINVAL, "slab_power_step: y and v ghosts come in pairs");
  int rc = use_device(h);
  if (rc) return rc;
  const int nb = emrkc_k::power_blocks();
  const int a = h->sp_a;
  CK(h, emrkc_k::launch_power(h->geom, h->sp_code, h->buf[h->cur], h->sp_v[a], q, h->sp_fy,
                              stim_rate_at(&h->p, t), h->sp_v[1 - a], gy_lo, gy_hi, gv_lo,
                              gv_hi, h->d_red, nb, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  h->sp_a = 1 - a;
  return EMRKC_OK;
}

int emrkc_slab_power_end(emrkc_handle* h, double* v_out_slab) {
  if (!h) return set_global(EMRKC_EINVAL, "null handle");
  if (h->sp_code < 0) return set_err(h, EMRKC_ESTATE, "slab power iteration not begun");
  int rc = use_device(h);
  if (rc) return rc;
  if (v_out_slab)
    CK(h, cudaMemcpy(v_out_slab, h->sp_v[h->sp_a], sizeof(double) * h->len,
                     cudaMemcpyDeviceToHost));
  h->sp_code = -1;
  return EMRKC_OK;
}

