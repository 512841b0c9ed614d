// tests/cpp/shim_kats.cpp — the reference's scalar known-answer tests
// (P/tests/test_multirate.cpp:54-233, test_cheb.cpp:110-166,
// test_spectral.cpp:13-29, test_ionic.cpp:12-18) written against the C++
// shim (include/emrkc.hpp) exactly as the reference tests call mrkc::, so the
// generic integrator layer runs on the device. Prints one JSON line of
// named results for tests/test_cpp_shim.py.
#include <cmath>
#include <cstdio>
#include <string>

#include "emrkc.hpp"

using emrkc::SplitRhs;
using emrkc::Vec;

static SplitRhs scalar_split(double lF, double lS, double lE = 0.0, double yinf = 0.0) {
  SplitRhs rhs;  // P/tests/test_multirate.cpp:54-66
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

int main() {
  std::string js = "{";
  auto put = [&](const char* k, double v) {
    char b[96];
    std::snprintf(b, sizeof b, "%s\"%s\": %.17g", js.size() > 1 ? ", " : "", k, v);
    js += b;
  };
  try {
    // averaged_force_emrkc closed forms (:97-106, :124-131)
    put("af_m1", emrkc::averaged_force_emrkc(0.0, Vec{1.0}, 0.1, scalar_split(-10.0, -1.0, -5.0),
                                             1)[0]);
    put("af_exp", emrkc::averaged_force_emrkc(0.0, Vec{1.0}, 0.1, scalar_split(0.0, 0.0, -5.0),
                                              1)[0]);
    // averaged_force_mrkc m = 1 (:70-74)
    put("afm_m1", emrkc::averaged_force_mrkc(0.0, Vec{1.0}, 0.1, scalar_split(-10.0, -1.0), 1)[0]);
    // counters (:141-150)
    emrkc::EvalCounters ctr;
    SplitRhs rc = scalar_split(-10.0, -1.0, -2.0);
    rc.counters = &ctr;
    emrkc::averaged_force_emrkc(0.0, Vec{1.0}, 0.1, rc, 3);
    put("n_fF", (double)ctr.n_fF);
    put("n_fS", (double)ctr.n_fS);
    put("n_exp", (double)ctr.n_exp_steps);
    // rkc_iteration: s = 1 damped Euler and R_2 at eps = 0 (test_cheb.cpp:118-131)
    const emrkc::RhsFn lin4 = [](double, const Vec& y, Vec& o) { o[0] = -4.0 * y[0]; };
    put("rkc_s1", emrkc::rkc_iteration(0.0, Vec{2.0}, 0.3, lin4, 1, 0.05)[0]);
    put("R2", emrkc::stability_poly(2, 0.0, -1.0));
    // non-finite stage names stage 1 (:139-149)
    int abort_stage = -1;
    try {
      const emrkc::RhsFn bad = [](double, const Vec&, Vec& o) { o.assign(o.size(), INFINITY); };
      emrkc::rkc_iteration(0.0, Vec{1.0}, 1.0, bad, 3, 0.05);
    } catch (const emrkc::NumericalAbort& e) {
      abort_stage = e.stage;
    }
    put("abort_stage", abort_stage);
    // gating-only emrkc_step, eps = 0, s = m = 1: exact exponential (:215-228)
    emrkc::MultirateStepReport rep;
    put("gating", emrkc::emrkc_step(0.0, Vec{1.0}, 0.8, scalar_split(0.0, 0.0, -4.0, 0.25), 0.0,
                                    emrkc::EmrkcVariant::standard, &rep)[0]);
    put("gating_s", rep.s);
    put("gating_m", rep.m);
    // missing exp_part is rejected (:229-233)
    int rejected = 0;
    try {
      SplitRhs r = scalar_split(-1.0, -1.0);
      r.exp_part = nullptr;
      emrkc::emrkc_step(0.0, Vec{1.0}, 0.1, r);
    } catch (const std::invalid_argument&) {
      rejected = 1;
    }
    put("rejected", rejected);
    // power iteration on diag(-3, -7) (test_spectral.cpp:21-29)
    const emrkc::RhsFn diag = [](double, const Vec& y, Vec& o) {
      o[0] = -3.0 * y[0];
      o[1] = -7.0 * y[1];
    };
    const auto est = emrkc::estimate_spectral_radius(0.0, Vec{0.5, 0.5}, diag, Vec{1.0, 1.0});
    put("rho_diag", est.rho / est.safety);
    // IonicModel adapter (test_ionic.cpp:12-18) and the resting state
    const auto hh = emrkc::make_ionic_model("hh");
    double a[3], b[3];
    hh->rates(-40.0, a, b);
    put("alpha_m_m40", a[0]);
    hh->rates(-55.0, a, b);
    put("alpha_n_m55", a[2]);
    const auto rest = hh->resting_state();
    put("V_rest", rest.V);
    put("I_rest", hh->ionic_current(rest.V, rest.z_E, {}));
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 1;
  }
  std::printf("%s}\n", js.c_str());
  return 0;
}
