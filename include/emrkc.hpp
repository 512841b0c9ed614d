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
//   RhsFn, SplitRhs, EvalCounters      P/include/mrkc/core.hpp:14,34-57,
//                                      multirate.hpp:25-35 (host callbacks)
//   rkc_iteration / stability_poly     P/include/mrkc/cheb.hpp:60-63,71-73
//   exponential_euler_step             P/include/mrkc/multirate.hpp:19-20
//   averaged_force_emrkc / _mrkc       P/include/mrkc/multirate.hpp:57-67
//   emrkc_step / mrkc_step (SplitRhs)  P/include/mrkc/multirate.hpp:72-81
//   estimate_spectral_radius (RhsFn)   P/include/mrkc/spectral.hpp:28-29
//   IonicModel / make_hh_model         P/include/mrkc/ionic.hpp:17-61
//   bind_split_rhs(DeviceMonodomain&)  the device operator as a SplitRhs
//
// The generic functions run the reference's recurrences on the device
// (include/emrkc.h, emrkc_generic.cu); a host RhsFn is called with its
// argument read back from the device and its result uploaded, so any
// reference-style callback works, and bind_split_rhs() keeps the
// monodomain operator's callbacks on the device.
//
// Header-only; link libemrkc_b200.so. Errors follow the reference:
// std::invalid_argument for bad arguments, NumericalAbort for non-finite
// stages, std::runtime_error for device failures.
#pragma once

#include <algorithm>
#include <exception>
#include <functional>
#include <memory>
#include <span>
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
                            const emrkc_partition* part = nullptr)
      : p_(p), part_(part ? *part : emrkc_partition{0, p.n[p.dim - 1]}) {
    check(emrkc_create(&p, device, part, &h_));
  }
  ~DeviceMonodomain() { emrkc_destroy(h_); }
  DeviceMonodomain(const DeviceMonodomain&) = delete;
  DeviceMonodomain& operator=(const DeviceMonodomain&) = delete;
  DeviceMonodomain(DeviceMonodomain&& o) noexcept : p_(o.p_), part_(o.part_), h_(o.h_) {
    o.h_ = nullptr;
  }

  emrkc_handle* handle() const { return h_; }
  int64_t size() const { return emrkc_local_len(h_); }

  // Uniform resting state (P/src/monodomain.cpp:306-319) of this handle's
  // slab: [V | gates | aux] (aux for EMRKC_MODEL_HH_AUX).
  Vec initial_state() const {
    const int64_t glen = emrkc_state_len(&p_, nullptr);
    Vec g(glen);
    check(emrkc_initial_state(&p_, g.data(), glen));
    const int64_t nz = p_.n[p_.dim - 1], gnn = glen / fields(), plane = gnn / nz;
    const int64_t a = part_.z_begin * plane, n = (part_.z_end - part_.z_begin) * plane;
    Vec y(static_cast<size_t>(fields() * n));
    for (int64_t f = 0; f < fields(); ++f)
      std::copy(g.begin() + f * gnn + a, g.begin() + f * gnn + a + n, y.begin() + f * n);
    return y;
  }
  int64_t fields() const { return 4 + (p_.model == EMRKC_MODEL_HH_AUX ? p_.n_aux : 0); }

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
  emrkc_problem p_{};
  emrkc_partition part_{};
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

// ===========================================================================
// Generic integrator layer (P/include/mrkc/cheb.hpp, multirate.hpp,
// spectral.hpp) over the C ABI's device implementation.
// ===========================================================================
using RhsFn = std::function<void(double t, const Vec& y, Vec& out)>;

struct EvalCounters {
  long long n_fF = 0, n_fS = 0, n_exp_steps = 0;
};

// SplitRhs over host callbacks (P/include/mrkc/multirate.hpp:25-35).
struct SplitRhs {
  RhsFn f_F;
  RhsFn f_S;
  std::function<void(const Vec& y, Vec& lambda, Vec& y_inf)> exp_part;
  double rho_F = 0.0;
  double rho_S = 0.0;
  EvalCounters* counters = nullptr;
  // set by bind_split_rhs: the device operator's own callbacks
  emrkc_split_rhs device{};
  bool on_device = false;
};

namespace detail {

// One context per host thread (device 0), like the reference's free functions.
inline emrkc_vctx* ctx() {
  struct Holder {
    emrkc_vctx* c = nullptr;
    ~Holder() { emrkc_vctx_destroy(c); }
  };
  thread_local Holder h;
  if (!h.c && emrkc_vctx_create(0, &h.c) != EMRKC_OK)
    throw std::runtime_error("emrkc: no usable CUDA device (there is no CPU fallback)");
  return h.c;
}

inline void vcheck(int rc, long stage = -1) {
  if (rc == EMRKC_OK) return;
  const std::string msg = emrkc_vctx_last_error(ctx());
  if (rc == EMRKC_EINVAL) throw std::invalid_argument(msg);
  if (rc == EMRKC_ENONFINITE) throw NumericalAbort(msg, -1, 0.0, static_cast<int>(stage));
  throw std::runtime_error(msg);
}

// RAII device vector of the context.
struct DVec {
  double* p = nullptr;
  int64_t n = 0;
  explicit DVec(int64_t n_) : n(n_) { vcheck(emrkc_vctx_alloc(ctx(), n, &p)); }
  DVec(const Vec& v) : DVec(static_cast<int64_t>(v.size())) {
    vcheck(emrkc_vctx_upload(ctx(), p, v.data(), n));
  }
  ~DVec() { emrkc_vctx_free(ctx(), p); }
  DVec(const DVec&) = delete;
  DVec& operator=(const DVec&) = delete;
  Vec host() const {
    Vec v(n);
    vcheck(emrkc_vctx_download(ctx(), v.data(), p, n));
    return v;
  }
};

struct HostRhs {
  const RhsFn* f;
  std::exception_ptr err;  // what the callback threw (rethrown by the caller)
};
inline int host_rhs(void* c, double t, const double* y, double* out, int64_t len, void*) {
  auto* r = static_cast<HostRhs*>(c);
  try {
    Vec yy(len), oo(len, 0.0);
    if (emrkc_vctx_download(ctx(), yy.data(), y, len)) return 1;
    (*r->f)(t, yy, oo);
    if (static_cast<int64_t>(oo.size()) != len) return 1;
    return emrkc_vctx_upload(ctx(), out, oo.data(), len) ? 1 : 0;
  } catch (...) {
    r->err = std::current_exception();
    return 1;
  }
}

struct HostSplit {
  const SplitRhs* rhs;
  HostRhs fF, fS;
  std::exception_ptr err;  // thrown by exp_part
  emrkc_counters ctr{};
  emrkc_split_rhs c{};
};
inline int host_exp(void* cx, const double* y, double* lam, double* yinf, int64_t len, void*) {
  auto* h = static_cast<HostSplit*>(cx);
  try {
    Vec yy(len), l(len, 0.0), yi(len, 0.0);
    if (emrkc_vctx_download(ctx(), yy.data(), y, len)) return 1;
    h->rhs->exp_part(yy, l, yi);
    if (emrkc_vctx_upload(ctx(), lam, l.data(), len)) return 1;
    return emrkc_vctx_upload(ctx(), yinf, yi.data(), len) ? 1 : 0;
  } catch (...) {
    h->err = std::current_exception();
    return 1;
  }
}
inline void make_split(const SplitRhs& rhs, HostSplit& hs) {
  hs.rhs = &rhs;
  if (rhs.on_device) {
    hs.c = rhs.device;
  } else {
    hs.fF.f = &rhs.f_F;
    hs.fS.f = &rhs.f_S;
    hs.c.f_F = rhs.f_F ? host_rhs : nullptr;
    hs.c.f_F_ctx = &hs.fF;
    hs.c.f_S = rhs.f_S ? host_rhs : nullptr;
    hs.c.f_S_ctx = &hs.fS;
    hs.c.exp_part = rhs.exp_part ? host_exp : nullptr;
    hs.c.exp_ctx = &hs;
  }
  hs.c.rho_F = rhs.rho_F;
  hs.c.rho_S = rhs.rho_S;
  hs.c.counters = &hs.ctr;
}
inline void fold(const SplitRhs& rhs, const HostSplit& hs) {
  // a callback's own exception wins over the ECALLBACK status it caused
  for (const std::exception_ptr& e : {hs.fF.err, hs.fS.err, hs.err})
    if (e) std::rethrow_exception(e);
  if (!rhs.counters) return;
  rhs.counters->n_fF += hs.ctr.n_fF;
  rhs.counters->n_fS += hs.ctr.n_fS;
  rhs.counters->n_exp_steps += hs.ctr.n_exp_steps;
}

}  // namespace detail

// rkc_iteration(t, y, dt, f, s, epsilon) — P/src/cheb.cpp:84-105
inline Vec rkc_iteration(double t, const Vec& y, double dt, const RhsFn& f, int s,
                         double epsilon) {
  detail::DVec dy(y), out(static_cast<int64_t>(y.size()));
  detail::HostRhs hr{&f, {}};
  int32_t st = 0;
  const int rc = emrkc_rkc_iteration(detail::ctx(), t, dy.p, dy.n, dt, detail::host_rhs, &hr, s,
                                     epsilon, out.p, &st);
  if (hr.err) std::rethrow_exception(hr.err);  // the callback's own exception
  detail::vcheck(rc, st);
  return out.host();
}
inline Vec rkc_iteration(double t, const Vec& y, double dt, const RhsFn& f, const RkcCoeffs& k) {
  return rkc_iteration(t, y, dt, f, k.s, k.epsilon);
}

// stability_poly(s, eps, z) — P/src/cheb.cpp:114-118
inline double stability_poly(int s, double epsilon, double z) {
  const RhsFn f = [z](double, const Vec& u, Vec& out) { out[0] = z * u[0]; };
  return rkc_iteration(0.0, Vec{1.0}, 1.0, f, s, epsilon)[0];
}

// exponential_euler_step — P/src/multirate.cpp:49-58
inline Vec exponential_euler_step(const Vec& y, double eta, const Vec& lambda_diag,
                                  const Vec& y_inf) {
  if (lambda_diag.size() != y.size() || y_inf.size() != y.size())
    throw std::invalid_argument("exponential_euler_step: size mismatch");
  detail::DVec dy(y), dl(lambda_diag), di(y_inf), out(static_cast<int64_t>(y.size()));
  detail::vcheck(emrkc_exponential_euler(detail::ctx(), dy.p, eta, dl.p, di.p, dy.n, out.p));
  return out.host();
}

// averaged_force_emrkc / averaged_force_mrkc — P/src/multirate.cpp:60-119
inline Vec averaged_force_emrkc(double t, const Vec& y, double eta, const SplitRhs& rhs, int m,
                                EmrkcVariant variant = EmrkcVariant::standard,
                                double epsilon = 0.05) {
  detail::DVec dy(y), out(static_cast<int64_t>(y.size()));
  detail::HostSplit hs;
  detail::make_split(rhs, hs);
  int32_t st = 0;
  const int rc = emrkc_averaged_force(detail::ctx(), t, dy.p, dy.n, eta, &hs.c, m,
                                      static_cast<int32_t>(variant), epsilon, out.p, &st);
  detail::fold(rhs, hs);
  detail::vcheck(rc, st);
  return out.host();
}
inline Vec averaged_force_mrkc(double t, const Vec& y, double eta, const SplitRhs& rhs, int m,
                               double epsilon = 0.05) {
  detail::DVec dy(y), out(static_cast<int64_t>(y.size()));
  detail::HostSplit hs;
  detail::make_split(rhs, hs);
  int32_t st = 0;
  const int rc = emrkc_averaged_force_mrkc(detail::ctx(), t, dy.p, dy.n, eta, &hs.c, m, epsilon,
                                           out.p, &st);
  detail::fold(rhs, hs);
  detail::vcheck(rc, st);
  return out.host();
}

// emrkc_step / mrkc_step over a SplitRhs — P/src/multirate.cpp:158-189
inline Vec emrkc_step(double t, const Vec& y, double dt, const SplitRhs& rhs,
                      double epsilon = 0.05, EmrkcVariant variant = EmrkcVariant::standard,
                      MultirateStepReport* report = nullptr) {
  detail::DVec dy(y), out(static_cast<int64_t>(y.size()));
  detail::HostSplit hs;
  detail::make_split(rhs, hs);
  emrkc_step_report r{};
  const int rc = emrkc_step_split(detail::ctx(), t, dy.p, dy.n, dt, &hs.c, epsilon,
                                  static_cast<int32_t>(variant), out.p, &r);
  detail::fold(rhs, hs);
  if (report) *report = DeviceMonodomain::to_report(r);
  detail::vcheck(rc, r.abort_stage);
  return out.host();
}
inline Vec mrkc_step(double t, const Vec& y, double dt, const SplitRhs& rhs,
                     double epsilon = 0.05, MultirateStepReport* report = nullptr) {
  detail::DVec dy(y), out(static_cast<int64_t>(y.size()));
  detail::HostSplit hs;
  detail::make_split(rhs, hs);
  emrkc_step_report r{};
  const int rc =
      emrkc_mrkc_step_split(detail::ctx(), t, dy.p, dy.n, dt, &hs.c, epsilon, out.p, &r);
  detail::fold(rhs, hs);
  if (report) *report = DeviceMonodomain::to_report(r);
  detail::vcheck(rc, r.abort_stage);
  return out.host();
}

// estimate_spectral_radius(t, y, f, v0, rho0) — P/src/spectral.cpp:26-71
struct RhoEstimateV {
  double rho = 0.0;
  Vec v;
  int iterations = 0;
  double safety = 1.05;
  bool converged = true;
};
inline RhoEstimateV estimate_spectral_radius(double t, const Vec& y, const RhsFn& f,
                                             const Vec& v0 = {}, double rho0 = 0.0) {
  detail::DVec dy(y), dv(static_cast<int64_t>(y.size()));
  std::unique_ptr<detail::DVec> d0;
  if (!v0.empty()) d0 = std::make_unique<detail::DVec>(v0);
  detail::HostRhs hr{&f, {}};
  emrkc_rho_result r{};
  const int rc = emrkc_estimate_spectral_radius(detail::ctx(), t, dy.p, dy.n, detail::host_rhs,
                                                &hr, d0 ? d0->p : nullptr, rho0, &r, dv.p);
  if (hr.err) std::rethrow_exception(hr.err);
  detail::vcheck(rc);
  RhoEstimateV e;
  e.rho = r.rho;
  e.iterations = r.iterations;
  e.safety = r.safety;
  e.converged = r.converged != 0;
  e.v = dv.host();
  return e;
}

// The device operator as a SplitRhs (callbacks stay on the device): the
// generic emrkc_step above then runs the grid problem.
inline SplitRhs bind_split_rhs(DeviceMonodomain& op, double rho_F = 0.0, double rho_S = 0.0) {
  SplitRhs r;
  check(emrkc_bind_split_rhs(op.handle(), &r.device), op.handle());
  r.on_device = true;
  r.rho_F = rho_F;
  r.rho_S = rho_S;
  return r;
}

// ===========================================================================
// IonicModel (P/include/mrkc/ionic.hpp:17-53) and the HH adapter over the
// library's model formulas (bit-identical to P/src/ionic.cpp:86-116).
// ===========================================================================
class IonicModel {
 public:
  virtual ~IonicModel() = default;
  virtual std::string name() const = 0;
  virtual int n_gates() const = 0;
  virtual int n_aux() const = 0;
  virtual std::vector<std::string> var_names() const = 0;
  virtual void rates(double V, std::span<double> alpha, std::span<double> beta) const = 0;
  virtual double ionic_current(double V, std::span<const double> z_E,
                               std::span<const double> z_S) const = 0;
  virtual void aux_rates(double, std::span<const double>, std::span<const double>,
                         std::span<double>) const {}
  struct Rest {
    double V = 0.0;
    Vec z_E;
    Vec z_S;
  };
  virtual Rest resting_state() const = 0;
  // lambda = -(alpha + beta), z_inf = alpha / (alpha + beta) (P/src/ionic.cpp:31-40)
  void gate_coeffs(double V, std::span<double> lambda, std::span<double> z_inf) const {
    std::vector<double> a(n_gates()), b(n_gates());
    rates(V, a, b);
    for (int g = 0; g < n_gates(); ++g) {
      lambda[g] = -(a[g] + b[g]);
      z_inf[g] = a[g] / (a[g] + b[g]);
    }
  }
  // The library model id the device kernels implement (EMRKC_MODEL_*).
  virtual int32_t model_id() const = 0;
};

class HodgkinHuxley final : public IonicModel {
 public:
  std::string name() const override { return "hh"; }
  int n_gates() const override { return 3; }
  int n_aux() const override { return 0; }
  std::vector<std::string> var_names() const override { return {"m", "h", "n"}; }
  void rates(double V, std::span<double> alpha, std::span<double> beta) const override {
    if (alpha.size() < 3 || beta.size() < 3) throw std::invalid_argument("hh: 3 gates");
    check(emrkc_model_rates(EMRKC_MODEL_HH, V, alpha.data(), beta.data()));
  }
  double ionic_current(double V, std::span<const double> z_E,
                       std::span<const double>) const override {
    if (z_E.size() < 3) throw std::invalid_argument("hh: 3 gates");
    double I = 0.0;
    check(emrkc_model_ionic_current(EMRKC_MODEL_HH, V, z_E.data(), &I));
    return I;
  }
  Rest resting_state() const override {
    Rest r;
    r.z_E.resize(3);
    check(emrkc_resting_state(EMRKC_MODEL_HH, &r.V, r.z_E.data()));
    return r;
  }
  int32_t model_id() const override { return EMRKC_MODEL_HH; }
};

inline std::unique_ptr<IonicModel> make_hh_model() { return std::make_unique<HodgkinHuxley>(); }

// make_ionic_model(name) (P/src/ionic.cpp:125-128): "hh" only.
inline std::unique_ptr<IonicModel> make_ionic_model(const std::string& name) {
  if (name == "hh") return make_hh_model();
  throw std::invalid_argument("unknown ionic model '" + name + "'");
}

}  // namespace emrkc
