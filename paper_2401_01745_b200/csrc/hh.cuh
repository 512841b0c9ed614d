// hh.cuh — Hodgkin–Huxley ionic model on the device (fp64).
//
// Restates HodgkinHuxley::rates / ionic_current (P/src/ionic.cpp:80-116),
// IonicModel::gate_coeffs (:31-40) and lin_exp_ratio (:14-21).
//
// Two evaluation strategies, selected at compile time by the kernels:
//  * hh_ref_*  : the reference's evaluation order, one exp per rate and IEEE
//                divisions (6 exp + 9 div per node). Used by the operator
//                evaluations (f_S in the power iteration) where the result is
//                differenced against a 1e-8 perturbation.
//  * hh_fast_* : the same functions with shared transcendental work:
//                exp(-(V+35)/10) = e^{1/2} exp(-(V+40)/10),
//                exp(-(V+55)/10) = e^{-3/2} exp(-(V+40)/10),
//                exp(-(V+65)/20) = exp(-(V+65)/80)^4,
//                so 3 exps instead of 6, and the six divisions are folded into
//                one reciprocal (Montgomery batch inversion). Each rewrite
//                changes results by a few ulp (<1e-14 relative), far inside the
//                rel-L2 <= 1e-9 parity bound of north_star.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>

namespace emrkc_dev {

// HH constants — P/src/ionic.cpp:86-91 (mS/mm^2, mV)
constexpr double kGNa = 1.2;
constexpr double kGK = 0.36;
constexpr double kGLeak = 0.003;
constexpr double kVNa = 50.0;
constexpr double kVK = -77.0;
constexpr double kVLeak = -54.387;

// ---------------------------------------------------------------------------
// Reference-order evaluation
// ---------------------------------------------------------------------------
__device__ __forceinline__ double lin_exp_ratio_ref(double x, double k) {
  const double u = x / k;
  if (fabs(u) < 1e-4) return k * (1.0 + u * (0.5 + u / 12.0));
  return x / (1.0 - exp(-u));
}

__device__ __forceinline__ void hh_rates_ref(double V, double* a, double* b) {
  a[0] = 0.1 * lin_exp_ratio_ref(V + 40.0, 10.0);
  b[0] = 4.0 * exp(-(V + 65.0) / 18.0);
  a[1] = 0.07 * exp(-(V + 65.0) / 20.0);
  b[1] = 1.0 / (1.0 + exp(-(V + 35.0) / 10.0));
  a[2] = 0.01 * lin_exp_ratio_ref(V + 55.0, 10.0);
  b[2] = 0.125 * exp(-(V + 65.0) / 80.0);
}

__device__ __forceinline__ void hh_gate_coeffs_ref(double V, double* lam,
                                                   double* zinf) {
  double a[3], b[3];
  hh_rates_ref(V, a, b);
#pragma unroll
  for (int g = 0; g < 3; ++g) {
    lam[g] = -(a[g] + b[g]);
    zinf[g] = a[g] / (a[g] + b[g]);
  }
}

// I_ion in the reference's left-to-right order (P/src/ionic.cpp:111-116).
__device__ __forceinline__ double hh_current(double V, double m, double h,
                                             double n) {
  const double ina = __dmul_rn(
      __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(kGNa, m), m), m), h), V - kVNa);
  const double ik = __dmul_rn(
      __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(kGK, n), n), n), n), V - kVK);
  const double il = __dmul_rn(kGLeak, V - kVLeak);
  return __dadd_rn(__dadd_rn(ina, ik), il);
}

// ---------------------------------------------------------------------------
// Shared-transcendental evaluation
// ---------------------------------------------------------------------------
// Gate coefficients of the three gates: lam = -(alpha+beta),
// zinf = alpha/(alpha+beta).
__device__ __forceinline__ void hh_gate_coeffs_fast(double V, double* lam,
                                                    double* zinf) {
  constexpr double kE05 = 1.6487212707001282;    // e^{0.5}
  constexpr double kEm15 = 0.22313016014842982;  // e^{-1.5}
  const double xm = V + 40.0;                    // alpha_m argument
  const double xn = V + 55.0;                    // alpha_n argument
  const double um = xm * 0.1;                    // x/10
  const double un = xn * 0.1;
  const double e10 = exp(-um);                   // exp(-(V+40)/10)
  const double w = -(V + 65.0);
  const double e18 = exp(w * (1.0 / 18.0));      // exp(-(V+65)/18)
  const double e80 = exp(w * 0.0125);            // exp(-(V+65)/80)
  const double e40 = e80 * e80;
  const double e20 = e40 * e40;                  // exp(-(V+65)/20)

  // alpha_m = 0.1 x/(1-e^{-x/10}); series 0.1*10*(1+u/2+u^2/12) for |u|<1e-4
  const bool sm = fabs(um) < 1e-4;
  const bool sn = fabs(un) < 1e-4;
  const double dm = sm ? 1.0 : 1.0 - e10;                 // denominators
  const double dn = sn ? 1.0 : 1.0 - e10 * kEm15;
  const double dh = 1.0 + e10 * kE05;
  const double nm = sm ? 1.0 + um * (0.5 + um * (1.0 / 12.0)) : 0.1 * xm;
  const double nn = sn ? 0.1 * (1.0 + un * (0.5 + un * (1.0 / 12.0))) : 0.01 * xn;

  const double bm = 4.0 * e18;
  const double ah = 0.07 * e20;
  const double bn = 0.125 * e80;

  // alpha+beta as fractions: s_m = (nm + bm dm)/dm etc.
  const double pm = nm + bm * dm;   // (alpha_m+beta_m) * dm
  const double pn = nn + bn * dn;   // (alpha_n+beta_n) * dn
  const double ph = ah * dh + 1.0;  // (alpha_h+beta_h) * dh
  // Batch inversion of dm, dn, dh, pm, pn, ph with one division.
  const double q1 = dm * dn;
  const double q2 = q1 * dh;
  const double q3 = q2 * pm;
  const double q4 = q3 * pn;
  const double q5 = q4 * ph;
  double r = 1.0 / q5;
  const double iph = r * q4;  r *= ph;
  const double ipn = r * q3;  r *= pn;
  const double ipm = r * q2;  r *= pm;
  const double idh = r * q1;  r *= dh;
  const double idn = r * dm;
  const double idm = r * dn;
  (void)idh;
  // lam = -(alpha+beta) = -p/d ; zinf = alpha/(alpha+beta) = numerator/p
  lam[0] = -(pm * idm);
  zinf[0] = nm * ipm;
  lam[1] = -(ph * idh);
  zinf[1] = (ah * dh) * iph;
  lam[2] = -(pn * idn);
  zinf[2] = nn * ipn;
}

// Reference-order exponential Euler of the gates (the fast kernels' path
// for V outside fast_math.cuh's window, or non-finite V): d = expm1(eta*Lambda)(z - z_inf).
struct Dgate {
  double d0, d1, d2;
};
static __device__ __noinline__ Dgate hh_expeuler_ref(double V, double z0, double z1,
                                                     double z2, double eta) {
  double lam[3], zinf[3];
  hh_gate_coeffs_ref(V, lam, zinf);
  Dgate d;
  d.d0 = expm1(eta * lam[0]) * (z0 - zinf[0]);
  d.d1 = expm1(eta * lam[1]) * (z1 - zinf[1]);
  d.d2 = expm1(eta * lam[2]) * (z2 - zinf[2]);
  return d;
}

}  // namespace emrkc_dev
