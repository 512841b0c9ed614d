// emrkc.hpp — C++ host shim over the C ABI (include/emrkc.h), mirroring the
// reference's mrkc:: interface for the emRKC path (P/ = /root/reference/proj):
//
//   get_stages / rkc_coeffs            P/include/mrkc/cheb.hpp:53-63
//   NumericalAbort                     P/include/mrkc/core.hpp:18-24
//   MultirateStepReport                P/include/mrkc/multirate.hpp:44-51
//   RhoEstimate                        P/include/mrkc/spectral.hpp:10-16
//   DeviceMonodomain                   MonodomainOperator + its SplitRhs
//                                      binding (P/include/mrkc/monodomain.hpp:119-176,
//                                      P/src/simulate.cpp:153-157), resident in HBM
//   emrkc_step(t, y, dt, op, ...)      P/include/mrkc/multirate.hpp:78-81
//   EmrkcVariant                       P/include/mrkc/multirate.hpp:37-40
//   DeviceMonodomain::run              the emRKC branch of run_simulation's loop
//                                      (P/src/simulate.cpp:176-229)
//   exex_rl_step / DeviceMonodomain::exex_run
//                                      P/src/baselines.cpp:192-210 and the
//                                      exex_rl branch of run_simulation
//
// Header-only; link libemrkc_b200.so. Errors follow the reference:
// std::invalid_argument for bad arguments, NumericalAbort for non-finite
// stages, std::runtime_error for device failures.
#pragma once

#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "emrkc.h"

namespace emrkc {

using Vec = std::vector<double>;

class NumericalAbort : public std::runtime_error {
 public:
  NumericalAbort(std::string what, long step, double dt, int stage = -1)
      : std::runtime_error(std::move(what)), step_index(step), dt(dt), stage(stage) {}
  long step_index = -1;
  double dt = 0.0;
  int stage = -1;
};

inline void check(int rc, const emrkc_handle* h = nullptr, long step = -1, double dt = 0.0,
                  int stage = -1) {
  if (rc == EMRKC_OK) return;
  const std::string msg = h ? emrkc_last_error(h) : emrkc_global_error();
  if (rc == EMRKC_EINVAL) throw std::invalid_argument(msg);
  if (rc == EMRKC_ENONFINITE) throw NumericalAbort(msg, step, dt, stage);
  throw std::runtime_error(msg);
}

enum class EmrkcVariant : int32_t {
  standard = EMRKC_VARIANT_STANDARD,
  progressive = EMRKC_VARIANT_PROGRESSIVE
};

struct StagePlan {
  int s = 1;
  double ell = 0.0;
  double beta = 0.0;
};

inline StagePlan get_stages(double dt, double rho, double epsilon) {
  StagePlan p;
  int32_t s = 0;
  check(emrkc_get_stages(dt, rho, epsilon, &s, &p.ell, &p.beta));
  p.s = s;
  return p;
}

struct RkcCoeffs {
  int s = 0;
  double epsilon = 0.0, omega0 = 0.0, omega1 = 0.0;
  Vec b, mu, nu, kappa, c;
};

inline RkcCoeffs rkc_coeffs(int s, double epsilon) {
  if (s < 1) throw std::invalid_argument("rkc_coeffs: s must be >= 1");
  RkcCoeffs k;
  k.s = s;
  k.epsilon = epsilon;
  k.b.resize(s + 1);
  k.mu.resize(s + 1);
  k.nu.resize(s + 1);
  k.kappa.resize(s + 1);
  k.c.resize(s + 1);
  check(emrkc_rkc_coeffs(s, epsilon, &k.omega0, &k.omega1, k.b.data(), k.mu.data(), k.nu.data(),
                         k.kappa.data(), k.c.data()));
  return k;
}

struct MultirateStepReport {
  int s = 0, m = 0;
  double eta = 0.0, ell_s = 0.0, ell_m = 0.0;
  long long n_fF = 0, n_fS = 0, n_exp_steps = 0;
};

struct RhoEstimate {
  double rho = 0.0;
  int iterations = 0;
  double safety = 1.05;
  bool converged = true;
};

struct RunResult {
  emrkc_run_result raw{};
  bool aborted() const { return raw.aborted != 0; }
};

// Device-resident monodomain operator (HH). Non-copyable, movable.
class DeviceMonodomain {
 public:
  explicit DeviceMonodomain(const emrkc_problem& p, int device = 0,
                            const emrkc_partition* part = nullptr) {
    check(emrkc_create(&p, device, part, &h_));
  }
  ~DeviceMonodomain() { emrkc_destroy(h_); }
  DeviceMonodomain(const DeviceMonodomain&) = delete;
  DeviceMonodomain& operator=(const DeviceMonodomain&) = delete;
  DeviceMonodomain(DeviceMonodomain&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }

  emrkc_handle* handle() const { return h_; }
  int64_t size() const { return emrkc_local_len(h_); }

  // Uniform resting state (P/src/monodomain.cpp:306-319).
  Vec initial_state() const {
    double V = 0.0, z[3];
    check(emrkc_resting_state(EMRKC_MODEL_HH, &V, z));
    const int64_t nn = size() / 4;
    Vec y(size());
    for (int64_t i = 0; i < nn; ++i) {
      y[i] = V;
      for (int g = 0; g < 3; ++g) y[(1 + g) * nn + i] = z[g];
    }
    return y;
  }

  void set_state(const Vec& y) { check(emrkc_set_state(h_, y.data(), (int64_t)y.size()), h_); }
  Vec get_state() const {
    Vec y(size());
    check(emrkc_get_state(h_, y.data(), (int64_t)y.size()), h_);
    return y;
  }

  // SplitRhs callbacks with the reference's signatures (host Vec in/out).
  void f_F(double t, const Vec& y, Vec& out) const { rhs(EMRKC_RHS_F, t, y, out); }
  void f_S(double t, const Vec& y, Vec& out) const { rhs(EMRKC_RHS_S, t, y, out); }
  void exp_part(const Vec& y, Vec& lambda, Vec& y_inf) const {
    lambda.resize(y.size());
    y_inf.resize(y.size());
    check(emrkc_exp_part(h_, y.data(), lambda.data(), y_inf.data(), (int64_t)y.size()), h_);
  }

  // estimate_spectral_radius on the current device state.
  RhoEstimate estimate_spectral_radius(int which, double t = 0.0) const {
    emrkc_rho_result r{};
    check(emrkc_estimate_rho(h_, which, t, nullptr, 0.0, &r, nullptr), h_);
    return {r.rho, r.iterations, r.safety, r.converged != 0};
  }

  // One step of the device state (y is not assigned on NumericalAbort).
  MultirateStepReport step(double t, double dt, double rho_F, double rho_S,
                           double epsilon = 0.05,
                           EmrkcVariant variant = EmrkcVariant::standard) {
    emrkc_step_report r{};
    const int rc = emrkc_step(h_, t, dt, epsilon, static_cast<int32_t>(variant), rho_F, rho_S, &r);
    check(rc, h_, -1, dt, r.abort_stage);
    return to_report(r);
  }

  // run_simulation's emRKC loop (t = step*dt, aborts, norm guard, gate range).
  RunResult run(long step0, long nsteps, double dt, double rho_F, double rho_S,
                double epsilon = 0.05, EmrkcVariant variant = EmrkcVariant::standard) {
    RunResult res;
    check(emrkc_run(h_, step0, nsteps, dt, epsilon, static_cast<int32_t>(variant), rho_F, rho_S,
                    &res.raw),
          h_);
    return res;
  }

  // mRKC with the stiff-gate split (gates in `mask` join f_F).
  void set_stiff_gates(int mask) { check(emrkc_set_stiff_gates(h_, mask), h_); }
  MultirateStepReport mrkc_step(double t, double dt, double rho_F, double rho_S,
                                double epsilon = 0.05) {
    emrkc_step_report r{};
    const int rc = emrkc_mrkc_step(h_, t, dt, epsilon, rho_F, rho_S, &r);
    check(rc, h_, -1, dt, r.abort_stage);
    return to_report(r);
  }
  RunResult mrkc_run(long step0, long nsteps, double dt, double rho_F, double rho_S,
                     double epsilon = 0.05) {
    RunResult res;
    check(emrkc_mrkc_run(h_, step0, nsteps, dt, epsilon, rho_F, rho_S, &res.raw), h_);
    return res;
  }

  // IMEX-RL with CgConfig (rel_tol, max_iters 0 = 10 sqrt(n) + 1, jacobi).
  long imex_step(double t, double dt, double rel_tol = 1e-8, long max_iters = 0,
                 bool jacobi = true) {
    emrkc_step_report r{};
    int64_t it = 0;
    check(emrkc_imex_step(h_, t, dt, rel_tol, max_iters, jacobi ? 1 : 0, &r, &it), h_, -1, dt);
    return static_cast<long>(it);
  }
  RunResult imex_run(long step0, long nsteps, double dt, double rel_tol = 1e-8,
                     long max_iters = 0, bool jacobi = true, long* cg_iters_total = nullptr) {
    RunResult res;
    int64_t it = 0;
    check(emrkc_imex_run(h_, step0, nsteps, dt, rel_tol, max_iters, jacobi ? 1 : 0, &res.raw,
                         &it),
          h_);
    if (cg_iters_total) *cg_iters_total = static_cast<long>(it);
    return res;
  }

  // rel_l2_error of SoA block `block` of the device state against host `ref`.
  double rel_l2_error(const Vec& ref, int block = 0) const {
    double e = 0.0;
    check(emrkc_rel_l2_error(h_, block, ref.data(), 0, &e), h_);
    return e;
  }

  // One EXEX-RL step of the device state (never throws NumericalAbort).
  void exex_step(double t, double dt) {
    emrkc_step_report r{};
    check(emrkc_exex_step(h_, t, dt, &r), h_);
  }

  // run_simulation's exex_rl loop (norm guard, gate range).
  RunResult exex_run(long step0, long nsteps, double dt) {
    RunResult res;
    check(emrkc_exex_run(h_, step0, nsteps, dt, &res.raw), h_);
    return res;
  }

  static MultirateStepReport to_report(const emrkc_step_report& r) {
    MultirateStepReport o;
    o.s = r.s;
    o.m = r.m;
    o.eta = r.eta;
    o.ell_s = r.ell_s;
    o.ell_m = r.ell_m;
    o.n_fF = r.n_fF;
    o.n_fS = r.n_fS;
    o.n_exp_steps = r.n_exp;
    return o;
  }

 private:
  void rhs(int which, double t, const Vec& y, Vec& out) const {
    out.resize(y.size());
    check(emrkc_eval_rhs(h_, which, t, y.data(), out.data(), (int64_t)y.size()), h_);
  }
  emrkc_handle* h_ = nullptr;
};

// Drop-in of `Vec emrkc_step(t, y, dt, rhs, epsilon, variant, report)`:
// host Vec in, one device step, host Vec out.
inline Vec emrkc_step(double t, const Vec& y, double dt, DeviceMonodomain& op, double rho_F,
                      double rho_S, double epsilon = 0.05,
                      MultirateStepReport* report = nullptr,
                      EmrkcVariant variant = EmrkcVariant::standard) {
  Vec out(y.size());
  emrkc_step_report r{};
  const int rc = emrkc_step_host(op.handle(), t, y.data(), out.data(), (int64_t)y.size(), dt,
                                 epsilon, static_cast<int32_t>(variant), rho_F, rho_S, &r);
  if (report) *report = DeviceMonodomain::to_report(r);
  check(rc, op.handle(), -1, dt, r.abort_stage);
  return out;
}

// Drop-in of `Vec exex_rl_step(t, y, dt, prob, counters)`
// (P/src/baselines.cpp:192-210): host Vec in, one device step, host Vec out.
inline Vec exex_rl_step(double t, const Vec& y, double dt, DeviceMonodomain& op) {
  op.set_state(y);
  op.exex_step(t, dt);
  return op.get_state();
}

}  // namespace emrkc
