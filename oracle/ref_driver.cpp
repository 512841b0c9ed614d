// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the
// product). A thin extern "C" harness, written for this repo, around the
// UNMODIFIED reference sources under /root/reference/proj/src, compiled
// together with them by oracle/Makefile into oracle/_ref/libmrkc_ref.so.
//
// It drives the reference exactly as its own run loop does
// (P/src/simulate.cpp:95-234, emRKC branch :151-163 and :197-228), except
// that it builds MonodomainOperator directly so that the conductivity,
// stimulus and the seeded initial state can be chosen (run_simulation
// hard-codes Conductivity::defaults(), P/src/simulate.cpp:28).
//
// Only tests/, __graft_entry__.smoke() and bench.py's reference /
// cpu_baseline legs load this library.

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <random>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "mrkc/baselines.hpp"
#include "mrkc/cheb.hpp"
#include "mrkc/ionic.hpp"
#include "mrkc/monodomain.hpp"
#include "mrkc/multirate.hpp"
#include "mrkc/spectral.hpp"

#include "emrkc.h"  // emrkc_problem / report structs (plain data only)

using namespace mrkc;

namespace {

thread_local std::string g_err;

// EMRKC_MODEL_HH_AUX (include/emrkc.h): the SYNTHETIC width stand-in, HH plus
// n_aux passive auxiliary variables, written here as an IonicModel of the
// reference's own interface (P/include/mrkc/ionic.hpp:17-53) so that the
// reference's generic machinery — StateLayout with n_aux, f_S aux rows
// (aux_rates_field, P/src/monodomain.cpp:191-221), exponential Euler passing
// aux through — runs it. Test infrastructure; no physiology.
class HHAux final : public IonicModel {
 public:
  explicit HHAux(int n_aux) : hh_(make_hh_model()), na_(n_aux) {}
  std::string name() const override { return "hh_aux"; }
  int n_gates() const override { return 3; }
  int n_aux() const override { return na_; }
  std::vector<std::string> var_names() const override {
    std::vector<std::string> v = {"m", "h", "n"};
    for (int a = 0; a < na_; ++a) v.push_back("aux" + std::to_string(a));
    return v;
  }
  void rates(double V, std::span<double> alpha, std::span<double> beta) const override {
    hh_->rates(V, alpha, beta);
  }
  double ionic_current(double V, std::span<const double> z_E,
                       std::span<const double>) const override {
    return hh_->ionic_current(V, z_E, {});
  }
  static double k(int a) { return 0.002 * static_cast<double>(1 + a % 5); }
  static double s1(int a) { return 0.01 * static_cast<double>(a % 3); }
  static double s0(int a) { return 0.5 + 0.1 * static_cast<double>(a % 4); }
  void aux_rates(double V, std::span<const double>, std::span<const double> z_S,
                 std::span<double> out) const override {
    for (int a = 0; a < na_; ++a) out[a] = k(a) * ((s1(a) * V + s0(a)) - z_S[a]);
  }
  Rest resting_state() const override {
    Rest r = hh_->resting_state();
    r.z_S.resize(na_);
    for (int a = 0; a < na_; ++a) r.z_S[a] = s1(a) * r.V + s0(a);
    return r;
  }

 private:
  std::unique_ptr<IonicModel> hh_;
  int na_;
};

std::unique_ptr<MonodomainOperator> make_op(const emrkc_problem* p) {
  if (p->model != EMRKC_MODEL_HH && p->model != EMRKC_MODEL_HH_AUX)
    throw ConfigError("unknown ionic model");
  if (p->model == EMRKC_MODEL_HH_AUX && (p->n_aux < 1 || p->n_aux > EMRKC_MAX_AUX))
    throw ConfigError("hh_aux: n_aux out of range");
  std::vector<double> extent(p->dim), dx(p->dim);
  for (int a = 0; a < p->dim; ++a) {
    dx[a] = p->dx[a];
    extent[a] = static_cast<double>(p->n[a] - 1) * p->dx[a];
  }
  Grid g = make_grid(p->dim, extent, dx);
  for (int a = 0; a < p->dim; ++a)
    if (g.n[a] != p->n[a]) throw ConfigError("grid: node count mismatch");
  Conductivity c;
  for (int a = 0; a < 3; ++a) c.sigma[a] = p->sigma[a];
  c.chi = p->chi;
  c.C_m = p->C_m;
  StimulusProtocol st;
  st.chi_amplitude = p->stim_chi_amplitude;
  for (int a = 0; a < 3; ++a) {
    st.box_lo[a] = p->stim_lo[a];
    st.box_hi[a] = p->stim_hi[a];
  }
  st.t_start = p->stim_t0;
  st.t_end = p->stim_t1;
  std::shared_ptr<const IonicModel> model;
  if (p->model == EMRKC_MODEL_HH_AUX)
    model = std::make_shared<HHAux>(p->n_aux);
  else
    model = make_hh_model();
  return std::make_unique<MonodomainOperator>(g, c, model, st);
}

SplitRhs bind(const MonodomainOperator& op, EvalCounters* ctr) {
  // Same lambdas as P/src/simulate.cpp:153-157.
  SplitRhs rhs;
  rhs.f_F = [&op](double t, const Vec& u, Vec& out) { op.f_F(t, u, out); };
  rhs.f_S = [&op](double t, const Vec& u, Vec& out) { op.f_S(t, u, out); };
  rhs.exp_part = [&op](const Vec& u, Vec& lam, Vec& yinf) {
    op.exp_part(u, lam, yinf);
  };
  rhs.counters = ctr;
  return rhs;
}

// Parses "... stage N" from the NumericalAbort message (P/src/cheb.cpp:76-78).
int stage_of(const char* what) {
  const char* k = std::strstr(what, "stage ");
  return k ? std::atoi(k + 6) : -1;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const NumericalAbort& e) {
    g_err = e.what();
    return EMRKC_ENONFINITE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return EMRKC_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return EMRKC_EINVAL;
  }
}

double max_abs_v(const Vec& y, long nn) {  // P/src/simulate.cpp:67-74
  double m = 0.0;
  for (long i = 0; i < nn; ++i) {
    if (!std::isfinite(y[i])) return std::numeric_limits<double>::infinity();
    m = std::max(m, std::abs(y[i]));
  }
  return m;
}

void track_gate_range(const Vec& y, const StateLayout& lay, double& lo,
                      double& hi) {  // P/src/simulate.cpp:76-85
  if (lay.n_gates == 0) return;
  const long begin = lay.gate_offset(0);
  const long end = begin + static_cast<long>(lay.n_gates) * lay.n_nodes;
  for (long k = begin; k < end; ++k) {
    lo = std::min(lo, y[k]);
    hi = std::max(hi, y[k]);
  }
}

std::vector<int> gates_of(int mask) {
  std::vector<int> g;
  for (int i = 0; i < 3; ++i)
    if (mask >> i & 1) g.push_back(i);
  return g;
}

// run_simulation's loop (P/src/simulate.cpp:176-229): method 0 emrkc,
// 1 emrkc_progressive (:197-207), 2 exex_rl (:211-212), 3 mrkc (:191-195)
// with the stiff-gate split of :132-150 (gates in `stiff`).
void run_loop(const MonodomainOperator& op, Vec& y, long step0, long nsteps,
              double dt, double eps, double rho_F, double rho_S,
              emrkc_run_result* res, double* wall_s, int method = 0, int stiff_mask = 0) {
  const StateLayout& lay = op.layout();
  EvalCounters ctr;
  SplitRhs rhs = bind(op, &ctr);
  if (method == 3) {
    const std::vector<int> stiff = gates_of(stiff_mask);
    rhs.f_F = [&op, stiff](double t, const Vec& u, Vec& out) {
      op.f_F_with_gates(stiff, t, u, out);
    };
    rhs.f_S = [&op, stiff](double t, const Vec& u, Vec& out) {
      op.f_S_with_gates(stiff, t, u, out);
    };
    rhs.exp_part = nullptr;
  }
  rhs.rho_F = rho_F;
  rhs.rho_S = rho_S;
  std::memset(res, 0, sizeof(*res));
  res->n_steps = nsteps;
  res->abort_step = -1;
  res->gate_min = 1.0;
  res->gate_max = 0.0;
  track_gate_range(y, lay, res->gate_min, res->gate_max);
  const auto w0 = std::chrono::steady_clock::now();
  for (long step = step0; step < step0 + nsteps; ++step) {
    const double t = static_cast<double>(step) * dt;
    try {
      if (method == 2) {
        y = exex_rl_step(t, y, dt, op, &ctr);
        res->s = res->m = 1;
        res->eta = dt;
      } else if (method == 3) {
        MultirateStepReport rep;
        y = mrkc_step(t, y, dt, rhs, eps, &rep);
        res->s = rep.s;
        res->m = rep.m;
        res->eta = rep.eta;
      } else {
        MultirateStepReport rep;
        y = emrkc_step(t, y, dt, rhs, eps,
                       method == 1 ? EmrkcVariant::progressive : EmrkcVariant::standard, &rep);
        res->s = rep.s;
        res->m = rep.m;
        res->eta = rep.eta;
      }
    } catch (const NumericalAbort& e) {
      res->aborted = 1;
      res->abort_kind = EMRKC_ABORT_NONFINITE;
      res->abort_step = step;
      res->abort_stage = stage_of(e.what());
      g_err = e.what();
      break;
    }
    ++res->steps_done;
    if (max_abs_v(y, lay.n_nodes) > 1e6) {
      res->aborted = 1;
      res->abort_kind = EMRKC_ABORT_NORM_GUARD;
      res->abort_step = step;
      break;
    }
    track_gate_range(y, lay, res->gate_min, res->gate_max);
  }
  const auto w1 = std::chrono::steady_clock::now();
  if (wall_s) *wall_s = std::chrono::duration<double>(w1 - w0).count();
  res->n_fF = ctr.n_fF;
  res->n_fS = ctr.n_fS;
  res->n_exp = ctr.n_exp_steps;
  res->device_ms = 0.0;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int64_t ref_state_len(const emrkc_problem* p) {
  int64_t nn = 1;
  for (int a = 0; a < p->dim; ++a) nn *= p->n[a];
  return nn * (4 + (p->model == EMRKC_MODEL_HH_AUX ? p->n_aux : 0));  // V + 3 gates + aux
}

int ref_resting_state(double* V, double* gates) {
  return guarded([&] {
    const auto hh = make_hh_model();
    const IonicModel::Rest r = hh->resting_state();
    *V = r.V;
    for (int g = 0; g < hh->n_gates(); ++g) gates[g] = r.z_E[g];
  });
}

int ref_hh_rates(double V, double* alpha, double* beta) {
  return guarded([&] {
    const auto hh = make_hh_model();
    hh->rates(V, std::span<double>(alpha, 3), std::span<double>(beta, 3));
  });
}

int ref_gate_coeffs(double V, double* lam, double* zinf) {
  return guarded([&] {
    const auto hh = make_hh_model();
    hh->gate_coeffs(V, std::span<double>(lam, 3), std::span<double>(zinf, 3));
  });
}

double ref_ionic_current(double V, const double* z) {
  const auto hh = make_hh_model();
  return hh->ionic_current(V, std::span<const double>(z, 3), {});
}

int ref_initial_state(const emrkc_problem* p, double* y) {
  return guarded([&] {
    const auto op = make_op(p);
    const Vec v = op->initial_state();
    std::memcpy(y, v.data(), v.size() * sizeof(double));
  });
}

int ref_rhs(const emrkc_problem* p, int which, double t, const double* y,
            double* out) {
  return guarded([&] {
    const auto op = make_op(p);
    const long len = op->layout().size();
    const Vec yv(y, y + len);
    Vec o;
    if (which == EMRKC_RHS_F)
      op->f_F(t, yv, o);
    else
      op->f_S(t, yv, o);
    std::memcpy(out, o.data(), len * sizeof(double));
  });
}

int ref_exp_part(const emrkc_problem* p, const double* y, double* lam,
                 double* yinf) {
  return guarded([&] {
    const auto op = make_op(p);
    const long len = op->layout().size();
    const Vec yv(y, y + len);
    Vec l, yi;
    op->exp_part(yv, l, yi);
    std::memcpy(lam, l.data(), len * sizeof(double));
    std::memcpy(yinf, yi.data(), len * sizeof(double));
  });
}

double ref_stimulus_rate(const emrkc_problem* p, double t, int64_t node) {
  const auto op = make_op(p);
  return op->stimulus_rate(t, node);
}

int ref_estimate_rho(const emrkc_problem* p, int which, double t,
                     const double* y, const double* v0, double rho0,
                     emrkc_rho_result* out, double* v_out) {
  return guarded([&] {
    const auto op = make_op(p);
    const long len = op->layout().size();
    const Vec yv(y, y + len);
    Vec v0v;
    if (v0) v0v.assign(v0, v0 + len);
    RhsFn f;
    const std::vector<int> stiff = gates_of((which >> 4) & 7);
    if ((which & 15) == EMRKC_RHS_F)
      f = [&](double tt, const Vec& u, Vec& o) { op->f_F(tt, u, o); };
    else if ((which & 15) == EMRKC_RHS_S)
      f = [&](double tt, const Vec& u, Vec& o) { op->f_S(tt, u, o); };
    else if ((which & 15) == 2)
      f = [&](double tt, const Vec& u, Vec& o) { op->f_F_with_gates(stiff, tt, u, o); };
    else
      f = [&](double tt, const Vec& u, Vec& o) { op->f_S_with_gates(stiff, tt, u, o); };
    const RhoEstimate est = estimate_spectral_radius(t, yv, f, v0v, rho0);
    out->rho = est.rho;
    out->iterations = est.iterations;
    out->converged = est.converged ? 1 : 0;
    out->safety = est.safety;
    if (v_out) std::memcpy(v_out, est.v.data(), len * sizeof(double));
  });
}

// Generic callback-operator power iteration, for the reference's own
// spectral KATs (P/tests/test_spectral.cpp) on small dense operators.
typedef void (*ref_rhs_cb)(double t, const double* y, double* out, int64_t n,
                           void* ctx);
int ref_estimate_rho_cb(ref_rhs_cb cb, void* ctx, int64_t n, double t,
                        const double* y, const double* v0, double rho0,
                        emrkc_rho_result* out, double* v_out) {
  return guarded([&] {
    const Vec yv(y, y + n);
    Vec v0v;
    if (v0) v0v.assign(v0, v0 + n);
    const RhsFn f = [&](double tt, const Vec& u, Vec& o) {
      o.resize(u.size());
      cb(tt, u.data(), o.data(), n, ctx);
    };
    const RhoEstimate est = estimate_spectral_radius(t, yv, f, v0v, rho0);
    out->rho = est.rho;
    out->iterations = est.iterations;
    out->converged = est.converged ? 1 : 0;
    out->safety = est.safety;
    if (v_out) std::memcpy(v_out, est.v.data(), n * sizeof(double));
  });
}

int ref_emrkc_step(const emrkc_problem* p, double t, const double* y,
                   double dt, double eps, double rho_F, double rho_S,
                   double* out, emrkc_step_report* rep) {
  std::memset(rep, 0, sizeof(*rep));
  const auto op = make_op(p);
  const long len = op->layout().size();
  EvalCounters ctr;
  SplitRhs rhs = bind(*op, &ctr);
  rhs.rho_F = rho_F;
  rhs.rho_S = rho_S;
  const Vec yv(y, y + len);
  const int rc = guarded([&] {
    MultirateStepReport r;
    const Vec o = emrkc_step(t, yv, dt, rhs, eps, EmrkcVariant::standard, &r);
    std::memcpy(out, o.data(), len * sizeof(double));
    rep->s = r.s;
    rep->m = r.m;
    rep->eta = r.eta;
    rep->ell_s = r.ell_s;
    rep->ell_m = r.ell_m;
  });
  rep->n_fF = ctr.n_fF;
  rep->n_fS = ctr.n_fS;
  rep->n_exp = ctr.n_exp_steps;
  if (rc == EMRKC_ENONFINITE) {
    rep->abort_kind = EMRKC_ABORT_NONFINITE;
    rep->abort_stage = stage_of(g_err.c_str());
  }
  return rc;
}

int ref_run(const emrkc_problem* p, double* y, int64_t step0, int64_t nsteps,
            double dt, double eps, double rho_F, double rho_S,
            emrkc_run_result* res, double* wall_s) {
  return guarded([&] {
    const auto op = make_op(p);
    const long len = op->layout().size();
    Vec yv(y, y + len);
    run_loop(*op, yv, step0, nsteps, dt, eps, rho_F, rho_S, res, wall_s);
    std::memcpy(y, yv.data(), len * sizeof(double));
  });
}

int ref_run_method(const emrkc_problem* p, double* y, int64_t step0, int64_t nsteps,
                   double dt, double eps, int32_t method, double rho_F, double rho_S,
                   emrkc_run_result* res, double* wall_s) {
  return guarded([&] {
    const auto op = make_op(p);
    const long len = op->layout().size();
    Vec yv(y, y + len);
    run_loop(*op, yv, step0, nsteps, dt, eps, rho_F, rho_S, res, wall_s, method & 15,
             (method >> 4) & 7);
    std::memcpy(y, yv.data(), len * sizeof(double));
  });
}

// run_simulation's imex_rl loop (P/src/simulate.cpp:176-229, :208-210)
int ref_run_imex(const emrkc_problem* p, double* y, int64_t step0, int64_t nsteps, double dt,
                 double rel_tol, int64_t max_iters, int32_t jacobi, emrkc_run_result* res,
                 int64_t* cg_iters_total) {
  return guarded([&] {
    const auto op = make_op(p);
    const StateLayout& lay = op->layout();
    const long len = lay.size();
    Vec yv(y, y + len);
    EvalCounters ctr;
    CgConfig cfg;
    cfg.rel_tol = rel_tol;
    cfg.max_iters = max_iters;
    cfg.preconditioner = jacobi ? CgConfig::Precond::jacobi : CgConfig::Precond::none;
    std::memset(res, 0, sizeof(*res));
    res->n_steps = nsteps;
    res->abort_step = -1;
    res->gate_min = 1.0;
    res->gate_max = 0.0;
    res->s = res->m = 1;
    res->eta = dt;
    track_gate_range(yv, lay, res->gate_min, res->gate_max);
    for (long step = step0; step < step0 + nsteps; ++step) {
      const double t = static_cast<double>(step) * dt;
      try {
        yv = imex_rl_step(t, yv, dt, *op, cfg, &ctr);
      } catch (const NumericalAbort& e) {
        res->aborted = 1;
        res->abort_kind = EMRKC_ABORT_NONFINITE;
        res->abort_step = step;
        res->abort_stage = -1;
        break;
      }
      ++res->steps_done;
      if (max_abs_v(yv, lay.n_nodes) > 1e6) {
        res->aborted = 1;
        res->abort_kind = EMRKC_ABORT_NORM_GUARD;
        res->abort_step = step;
        break;
      }
      track_gate_range(yv, lay, res->gate_min, res->gate_max);
    }
    res->n_fF = ctr.n_fF;
    res->n_fS = ctr.n_fS;
    res->n_exp = ctr.n_exp_steps;
    if (cg_iters_total) *cg_iters_total = ctr.cg_iters_total;
    std::memcpy(y, yv.data(), len * sizeof(double));
  });
}

int ref_identify_stiff_gates(const double* V, int64_t n, int32_t* order) {
  return guarded([&] {
    const auto model = make_hh_model();
    const std::vector<int> o = identify_stiff_gates(*model, std::span<const double>(V, n));
    for (std::size_t g = 0; g < o.size(); ++g) order[g] = o[g];
  });
}

int ref_rhs_gates(const emrkc_problem* p, int which, int stiff, double t, const double* y,
                  double* out) {
  return guarded([&] {
    const auto op = make_op(p);
    const long len = op->layout().size();
    const Vec yv(y, y + len);
    Vec o;
    const std::vector<int> s = gates_of(stiff);
    if (which == 0) op->f_F_with_gates(s, t, yv, o);
    else op->f_S_with_gates(s, t, yv, o);
    std::memcpy(out, o.data(), len * sizeof(double));
  });
}

// Reference-arm throughput: `nthreads` independent replicas of the
// reference's serial emRKC loop run concurrently (the reference has no
// intra-run parallelism; its only pool is over independent cells,
// P/src/experiments.cpp:22-37). Returns the per-replica loop seconds.
int ref_bench(const emrkc_problem* p, const double* y0, int64_t nsteps,
              double dt, double eps, double rho_F, double rho_S,
              int32_t nthreads, double* seconds) {
  return guarded([&] {
    const auto op = make_op(p);
    const long len = op->layout().size();
    std::vector<std::thread> th;
    std::vector<std::string> errs(nthreads);
    for (int k = 0; k < nthreads; ++k) {
      th.emplace_back([&, k] {
        try {
          Vec yv(y0, y0 + len);
          emrkc_run_result r;
          run_loop(*op, yv, 0, nsteps, dt, eps, rho_F, rho_S, &r,
                   &seconds[k]);
        } catch (const std::exception& e) {
          errs[k] = e.what();
        }
      });
    }
    for (auto& t : th) t.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
  });
}

double ref_rel_l2_error(const emrkc_problem* p, const double* a,
                        const double* b) {
  const auto op = make_op(p);
  const long nn = op->grid().n_nodes;
  try {
    return rel_l2_error(std::span<const double>(a, nn),
                        std::span<const double>(b, nn), op->grid());
  } catch (const std::exception& e) {
    g_err = e.what();
    return std::nan("");
  }
}

double ref_analytic_rho_F(const emrkc_problem* p) {
  const auto op = make_op(p);
  return analytic_rho_F(op->grid(), op->conductivity());
}

// ---- integrator layer on scalar surrogates (P/tests/test_multirate.cpp:54-66)

int ref_get_stages(double dt, double rho, double eps, int32_t* s, double* ell,
                   double* beta) {
  return guarded([&] {
    const StagePlan pl = get_stages(dt, rho, eps);
    *s = pl.s;
    *ell = pl.ell;
    *beta = pl.beta;
  });
}

int ref_rkc_coeffs(int32_t s, double eps, double* omega0, double* omega1,
                   double* b, double* mu, double* nu, double* kappa,
                   double* c) {
  return guarded([&] {
    const RkcCoeffs k = rkc_coeffs(s, eps);
    *omega0 = k.omega0;
    *omega1 = k.omega1;
    for (int j = 0; j <= s; ++j) {
      b[j] = k.b[j];
      mu[j] = k.mu[j];
      nu[j] = k.nu[j];
      kappa[j] = k.kappa[j];
      c[j] = k.c[j];
    }
  });
}

double ref_phi(double z) { return phi(z); }

int ref_rkc_iteration_scalar(double t, double y0, double dt, double lambda,
                             int32_t s, double eps, double* out) {
  return guarded([&] {
    const RhsFn f = [lambda](double, const Vec& y, Vec& o) {
      o[0] = lambda * y[0];
    };
    *out = rkc_iteration(t, Vec{y0}, dt, f, s, eps)[0];
  });
}

namespace {
SplitRhs scalar_split(double lF, double lS, double lE, double yinf) {
  SplitRhs rhs;  // same surrogate as P/tests/test_multirate.cpp:54-66
  rhs.f_F = [lF](double, const Vec& y, Vec& out) { out[0] = lF * y[0]; };
  rhs.f_S = [lS](double, const Vec& y, Vec& out) { out[0] = lS * y[0]; };
  rhs.exp_part = [lE, yinf](const Vec&, Vec& lam, Vec& yi) {
    lam[0] = lE;
    yi[0] = yinf;
  };
  rhs.rho_F = std::abs(lF);
  rhs.rho_S = std::abs(lS);
  return rhs;
}
}  // namespace

int ref_averaged_force_emrkc_scalar(double lF, double lS, double lE,
                                    double yinf, double y, double eta,
                                    int32_t m, double eps, double* out) {
  return guarded([&] {
    const SplitRhs rhs = scalar_split(lF, lS, lE, yinf);
    *out = averaged_force_emrkc(0.0, Vec{y}, eta, rhs, m,
                                EmrkcVariant::standard, eps)[0];
  });
}

int ref_emrkc_step_scalar(double lF, double lS, double lE, double yinf,
                          double y, double dt, double eps, double* out,
                          int32_t* s, int32_t* m, double* eta) {
  return guarded([&] {
    const SplitRhs rhs = scalar_split(lF, lS, lE, yinf);
    MultirateStepReport rep;
    *out = emrkc_step(0.0, Vec{y}, dt, rhs, eps, EmrkcVariant::standard,
                      &rep)[0];
    *s = rep.s;
    *m = rep.m;
    *eta = rep.eta;
  });
}

int ref_exponential_euler_step(const double* y, double eta, const double* lam,
                               const double* yinf, int64_t n, double* out) {
  return guarded([&] {
    const Vec o = exponential_euler_step(Vec(y, y + n), eta,
                                         Vec(lam, lam + n),
                                         Vec(yinf, yinf + n));
    std::memcpy(out, o.data(), n * sizeof(double));
  });
}

// libstdc++'s mt19937_64 + uniform_real_distribution(-1, 1): the generator
// the reference seeds its power-iteration direction with
// (P/src/spectral.cpp:16-22). Used to pin the C restatement's generator.
void ref_std_uniform_direction(uint64_t seed, int64_t n, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

void ref_std_normal(uint64_t seed, double mean, double sd, int64_t n,
                    double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist(mean, sd);
  for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

}  // extern "C"
