// fast_math.cuh — fp64 building blocks of the fast (default) kernels.
//
// The emRKC node update is FP64-pipe / issue bound on B200 once it is fused
// into one HBM pass (profiles/r01_v1_k_stage_m1.md: 79% issue, ~900 warp
// instructions per node with libdevice exp/expm1). These replacements keep
// full double accuracy (<= ~1.5 ulp) with far fewer instructions:
//  * exp_tab : table-driven exp, x = (256 k + j) ln2/256 + r, |r| <= ln2/512,
//              e^x = 2^k * T[j] * P4(r); T[j] = 2^(j/256) lives in shared
//              memory (2 KiB per block); 9 DP instructions + 1 LDS. Inputs
//              outside |x| < 700 (and NaN/Inf) take libdevice exp.
//  * rcp_fast: MUFU reciprocal seed + two Newton steps (4 DFMA).
#pragma once

#include <cuda_runtime.h>

#include "exp_table.cuh"

namespace emrkc_dev {

constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: round-to-int shifter

// fp64 constants whose low 32 bits are non-zero cannot be encoded as
// instruction immediates; keeping them in the constant bank lets every
// DFMA/DMUL read them as a c[][] operand instead of re-materialising them in
// registers (2 IMAD.MOV per use, seen in the r01 SASS).
struct FastConsts {
  double l2e256, ln2hi, ln2lo, c24, c6, c12;
  double p1, p01, p001, p07, p0125, r18, r80, e05, em15;
  double gna, gk, gl, vl;
  double e25;
};
__constant__ FastConsts kFC = {
    kL2E256, kLn2_256_hi, kLn2_256_lo, 1.0 / 24.0, 1.0 / 6.0, 1.0 / 12.0,
    0.1, 0.1, 0.01, 0.07, 0.125, 1.0 / 18.0, 0.0125, 1.6487212707001282,
    0.22313016014842982, 1.2, 0.36, 0.003, -54.387, 12.182493960703473};
// hh_expeuler_fast validity window (host: fast_window, per eta): every
// exp_tab_nc argument stays within +-700 and the batch product finite. The
// rates that grow without bound are beta_m = 4 e^{-(V+65)/18} (and
// beta_n) below rest and alpha_m ~ 0.1 (V + 40), alpha_n ~ 0.01 (V + 55)
// above it, so
//   V >= vlo(eta) >= -400: eta (alpha_g + beta_g) <= 580 for every gate,
//        solved on the host from the full sums (alpha_m adds ~0.4 to
//        beta_m near -56 mV; emrkc_capi.cpp fast_window) and verified by a
//        scan against 600; empty window (no fast nodes) if none exists
//   V <= min(10000, 6000 / eta - 80)         (eta (alpha_m + beta_m) <= 600)
// (at V = -400 the batch product is ~1e110, far from overflow; at 10000 the
// shared exponentials' arguments are ~ -560). Nodes outside the window (and
// non-finite V) take the reference-order path (hh_expeuler_ref). Before this
// window the bound was a fixed |V| <= 150 for eta <= 1.5: a strong stimulus
// pushed whole planes past +150 mV into the per-thread reference path.
// (kernels.h: fast_vlo / fast_vhi)

__device__ __forceinline__ double exp_tab(double x, const double* __restrict__ tab) {
  const int hi = __double2hiint(x);
  if ((hi & 0x7fffffff) >= 0x4085e000) return exp(x);  // |x| >= 700, NaN, Inf
  const double t = fma(x, kL2E256, kMagic);
  const int n = __double2loint(t);
  const double nd = t - kMagic;
  double r = fma(-nd, kLn2_256_hi, x);
  r = fma(-nd, kLn2_256_lo, r);
  // e^r, |r| <= 0.00136: Taylor to r^4 (truncation 3.8e-17 relative)
  double p = fma(r, 1.0 / 24.0, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double v = tab[n & 255] * p;  // in [1, 2.0001)
  return __hiloint2double(__double2hiint(v) + ((n >> 8) << 20), __double2loint(v));
}

// exp_tab without the range check: valid for -700 <= x <= 700 (the caller
// guarantees the range; see hh_expeuler_fast).
__device__ __forceinline__ double exp_tab_nc(double x, const double* __restrict__ tab) {
  const double t = fma(x, kFC.l2e256, kMagic);
  const int n = __double2loint(t);
  const double nd = t - kMagic;
  double r = fma(-nd, kFC.ln2hi, x);
  r = fma(-nd, kFC.ln2lo, r);
  double p = fma(r, kFC.c24, kFC.c6);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double v = tab[n & 255] * p;
  // 2^(n >> 8) into the exponent field: (n & ~255) << 12 == (n >> 8) << 20
  // (one LOP3 + one IMAD instead of a shift, a mask and an add)
  return __hiloint2double(__double2hiint(v) + (n & ~255) * 4096, __double2loint(v));
}

__device__ __forceinline__ double rcp_fast(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// Finite test on the high word only (integer pipe, not the FP64 pipe).
__device__ __forceinline__ bool finite_hi(double x) {
  return (__double2hiint(x) & 0x7ff00000) != 0x7ff00000;
}

// Fills the block's exp table (call before the block's first exp_tab and
// follow with __syncthreads()).
__device__ __forceinline__ void load_exp_table(double* sh, int tid, int nthreads) {
  for (int j = tid; j < 256; j += nthreads) sh[j] = kExp2Tab256[j];
}

// ---------------------------------------------------------------------------
// Valid inside the fast_vlo(eta) .. fast_vhi(eta) window (see above).
//
// Exponential Euler of the three HH gates at one node, with the rates
// evaluated through shared exponentials (hh.cuh, hh_gate_coeffs_fast) and
// one batch reciprocal:
//   y_E = z + expm1(eta Lambda(V)) (z - z_inf(V))     (P/src/multirate.cpp:49-58)
// Returns d = y_E - z per gate; y_E = z + d.
// expm1 is formed as exp_tab(x) - 1: x = eta*Lambda <= -eta*0.06, the
// subtraction is exact (Sterbenz) and the absolute error ~1e-16 enters the
// gate only through (z - z_inf), i.e. below one ulp of the gate.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void hh_expeuler_fast(double V, double z0, double z1,
                                                 double z2, double eta,
                                                 const double* __restrict__ tab,
                                                 double& d0, double& d1, double& d2) {
  const double xm = V + 40.0;
  const double xn = V + 55.0;
  const double um = xm * kFC.p1;
  const double un = xn * kFC.p1;
  const double w = -(V + 65.0);
  const double e18 = exp_tab_nc(w * kFC.r18, tab);  // exp(-(V+65)/18)
  const double e80 = exp_tab_nc(w * kFC.r80, tab);  // exp(-(V+65)/80)
  const double e40 = e80 * e80;
  const double e20 = e40 * e40;                     // exp(-(V+65)/20)
  // exp(-(V+40)/10) = exp(-(V+65)/80)^8 e^{2.5}: ~15 ulp, which reaches
  // alpha_m = 0.1 x/(1 - e10) amplified by 1/|x/10| <= 1e4 (series below
  // 1e-4): <= 2e-11 relative, and only within ~1 mV of V = -40.
  const double e10 = (e20 * e20) * kFC.e25;
  double dm = 1.0 - e10;
  double dn = fma(-e10, kFC.em15, 1.0);             // 1 - exp(-(V+55)/10)
  const double dh = fma(e10, kFC.e05, 1.0);         // 1 + exp(-(V+35)/10)
  double nm = kFC.p01 * xm;
  double nn = kFC.p001 * xn;
  // lin_exp_ratio's series branch (P/src/ionic.cpp:16-19): |x/10| < 1e-4,
  // i.e. V within 1e-3 mV of -40 or -55 — rare, kept out of the main path.
  if (fabs(um) < 1e-4 || fabs(un) < 1e-4) {
    if (fabs(um) < 1e-4) {
      dm = 1.0;
      nm = fma(um, fma(um, kFC.c12, 0.5), 1.0);
    }
    if (fabs(un) < 1e-4) {
      dn = 1.0;
      nn = kFC.p01 * fma(un, fma(un, kFC.c12, 0.5), 1.0);
    }
  }
  const double bm = 4.0 * e18;
  const double ahdh = (kFC.p07 * e20) * dh;
  const double bn = 0.125 * e80;
  const double pm = fma(bm, dm, nm);   // (alpha_m + beta_m) dm
  const double pn = fma(bn, dn, nn);   // (alpha_n + beta_n) dn
  const double ph = ahdh + 1.0;        // (alpha_h + beta_h) dh
  // one reciprocal for dm, dn, dh, pm, pn, ph (batch inversion as a
  // depth-3 tree: short dependency chain, 15 multiplies)
  const double A = dm * dn, B = dh * pm, C = pn * ph;
  const double AB = A * B;
  const double r = rcp_fast(AB * C);
  const double iAB = r * C, iC = r * AB;
  const double iA = iAB * B, iB = iAB * A;
  const double idm = iA * dn, idn = iA * dm;
  const double idh = iB * pm, ipm = iB * dh;
  const double ipn = iC * ph, iph = iC * pn;
  const double me = -eta;
  // eta*Lambda_g = -eta (alpha+beta) = -eta p/d >= -600 inside the window
  // (host-checked per node), so exp_tab_nc needs no clamp.
  const double em = exp_tab_nc(me * (pm * idm), tab) - 1.0;
  const double eh = exp_tab_nc(me * (ph * idh), tab) - 1.0;
  const double en = exp_tab_nc(me * (pn * idn), tab) - 1.0;
  d0 = em * (z0 - nm * ipm);
  d1 = eh * (z1 - ahdh * iph);
  d2 = en * (z2 - nn * ipn);
}

}  // namespace emrkc_dev
