// kernels.cu — sm_100a kernels of the emRKC monodomain step.
//
// Hot path: one outer RKC stage of emrkc_step
// (P/src/multirate.cpp:173-189) = exp_part + exponential Euler
// (P/src/monodomain.cpp:246-256, P/src/multirate.cpp:49-58), the frozen slow
// term f_S(y_E) (P/src/monodomain.cpp:214-221), the inner m-stage RKC
// iteration on f_F + f_S (P/src/cheb.cpp:84-105 over
// P/src/monodomain.cpp:73-90) and the outer three-term recurrence.
//
// Layout: the reference Vec, SoA fp64 [V | m | h | n], node index
// i0 + n0*(i1 + n1*i2). Threads map 32-wide onto axis 0 so every block load
// and store is a coalesced 256-byte row; the slab (slowest) axis may be
// partitioned, its neighbour planes then come from ghost buffers that the
// neighbour's kernels fill with peer stores (Halo::put_*).
//
// Rounding: the stencil and all RKC recurrences use explicit _rn intrinsics
// in the reference's evaluation order (no FMA contraction), so given equal
// inputs they are bit-identical to the reference; only the ionic
// transcendentals differ (ulp level), see hh.cuh.
#include <cfloat>
#include <climits>
#include <cstdio>

#include "aux.cuh"
#include "hh.cuh"
#include "kernels.h"

namespace emrkc_k {

using namespace emrkc_dev;

namespace {

constexpr int BX = 32;
constexpr int BY = 4;
constexpr int kThreads = BX * BY;

__device__ __forceinline__ bool finite(double x) { return isfinite(x); }

// Thread -> local node mapping (see file comment).
template <int DIM>
struct Node {
  int c0, c1, cz;     // local coordinates (cz along the slab axis)
  long long i, ip;    // local node index, index within the slab plane
  bool valid;
};

template <int DIM>
__device__ __forceinline__ Node<DIM> node_here(const Geom& g) {
  Node<DIM> n;
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (DIM == 3) {
    n.c0 = blockIdx.x * BX + tx;
    n.c1 = blockIdx.y * BY + ty;
    n.cz = blockIdx.z;
    n.valid = n.c0 < g.n0 && n.c1 < g.n1;
    n.ip = (long long)n.c0 + (long long)g.n0 * n.c1;
    n.i = n.ip + g.plane * n.cz;
  } else if (DIM == 2) {
    n.c0 = blockIdx.x * BX + tx;
    n.c1 = 0;
    n.cz = blockIdx.y * BY + ty;
    n.valid = n.c0 < g.n0 && n.cz < g.nzl;
    n.ip = n.c0;
    n.i = n.ip + g.plane * n.cz;
  } else {
    n.c0 = 0;
    n.c1 = 0;
    n.cz = (blockIdx.x * BY + ty) * BX + tx;
    n.valid = n.cz < g.nzl;
    n.ip = 0;
    n.i = n.cz;
  }
  return n;
}

template <int DIM>
__device__ __forceinline__ Node<DIM> node_flat(const Geom& g, long long i) {
  Node<DIM> n;
  n.i = i;
  n.valid = true;
  if (DIM == 3) {
    n.c0 = (int)(i % g.n0);
    const long long t = i / g.n0;
    n.c1 = (int)(t % g.n1);
    n.cz = (int)(t / g.n1);
    n.ip = i - g.plane * n.cz;
  } else if (DIM == 2) {
    n.c0 = (int)(i % g.n0);
    n.c1 = 0;
    n.cz = (int)(i / g.n0);
    n.ip = n.c0;
  } else {
    n.c0 = n.c1 = 0;
    n.cz = (int)i;
    n.ip = 0;
  }
  return n;
}

// Stimulus membership (P/src/monodomain.cpp:151-158) via the host-computed
// node box (the host evaluates the reference's x = i*dx comparison per axis).
template <int DIM>
__device__ __forceinline__ bool in_stim(const Geom& g, const Node<DIM>& n) {
  const int zg = n.cz + g.zoff;
  if (DIM == 3)
    return n.c0 >= g.st_lo[0] && n.c0 <= g.st_hi[0] && n.c1 >= g.st_lo[1] &&
           n.c1 <= g.st_hi[1] && zg >= g.st_lo[2] && zg <= g.st_hi[2];
  if (DIM == 2)
    return n.c0 >= g.st_lo[0] && n.c0 <= g.st_hi[0] && zg >= g.st_lo[1] &&
           zg <= g.st_hi[1];
  return zg >= g.st_lo[0] && zg <= g.st_hi[0];
}

// One axis term w*(vp - 2 v + vm) accumulated as the reference does
// (P/src/monodomain.cpp:85-87).
__device__ __forceinline__ double axis_term(double acc, double w, double vp,
                                            double vc, double vm) {
  return __dadd_rn(acc, __dmul_rn(w, __dadd_rn(__dsub_rn(vp, 2.0 * vc), vm)));
}

// Scaled Neumann Laplacian of a field at node n (diffusion_apply,
// P/src/monodomain.cpp:73-90): axes accumulated in order 0,1,2, mirror ghost
// at global boundaries, ghost planes at slab faces. F(j) returns the field
// at local index j, FL/FH(ip) the ghost plane values.
template <int DIM, class F, class FL, class FH>
__device__ __forceinline__ double lap(const Geom& g, const Node<DIM>& n,
                                      double vc, F f, FL flo, FH fhi) {
  double d = 0.0;
  if (DIM >= 2) {
    const double vm = (n.c0 > 0) ? f(n.i - 1) : f(n.i + 1);
    const double vp = (n.c0 < g.n0 - 1) ? f(n.i + 1) : f(n.i - 1);
    d = axis_term(d, g.w[0], vp, vc, vm);
  }
  if (DIM == 3) {
    const double vm = (n.c1 > 0) ? f(n.i - g.n0) : f(n.i + g.n0);
    const double vp = (n.c1 < g.n1 - 1) ? f(n.i + g.n0) : f(n.i - g.n0);
    d = axis_term(d, g.w[1], vp, vc, vm);
  }
  {
    const int zg = n.cz + g.zoff;
    const bool has_dn = n.cz > 0, has_up = n.cz + 1 < g.nzl;
    double vm, vp;
    if (zg > 0)
      vm = has_dn ? f(n.i - g.plane) : flo(n.ip);
    else
      vm = has_up ? f(n.i + g.plane) : fhi(n.ip);
    if (zg < g.nzg - 1)
      vp = has_up ? f(n.i + g.plane) : fhi(n.ip);
    else
      vp = has_dn ? f(n.i - g.plane) : flo(n.ip);
    d = axis_term(d, g.w[DIM - 1], vp, vc, vm);
  }
  return d;
}

struct Ld {
  const double* __restrict__ p;
  __device__ double operator()(long long j) const { return __ldg(p + j); }
};

// z = y + q v evaluated on the fly (power iteration, spectral.cpp:53)
struct LdZ {
  const double* __restrict__ y;
  const double* __restrict__ v;
  double q;
  __device__ double operator()(long long j) const {
    return __dadd_rn(y[j], __dmul_rn(q, v[j]));
  }
};

// Gate coefficients: fast or reference order.
template <int FAST>
__device__ __forceinline__ void gate_coeffs(double V, double* lam,
                                            double* zinf) {
  if (FAST)
    hh_gate_coeffs_fast(V, lam, zinf);
  else
    hh_gate_coeffs_ref(V, lam, zinf);
}

// y_E = y + expm1(eta*Lambda)(y - y_inf) — P/src/multirate.cpp:49-58.
__device__ __forceinline__ double exp_euler(double z, double eta, double lam,
                                            double zinf) {
  return __dadd_rn(z, __dmul_rn(expm1(__dmul_rn(eta, lam)), __dsub_rn(z, zinf)));
}

// V row of f_S — v_reaction, P/src/monodomain.cpp:160-173.
template <int FAST>
__device__ __forceinline__ double slow_v(const Geom& g, double stim, double V,
                                         double m, double h, double n) {
  const double I = hh_current(V, m, h, n);
  return __dsub_rn(stim, FAST ? __dmul_rn(I, g.inv_Cm) : __ddiv_rn(I, g.Cm));
}

// (u - g)/eta — P/src/multirate.cpp:117
template <int FAST>
__device__ __forceinline__ double avg_force(double u, double g0, double eta,
                                            double inv_eta) {
  return FAST ? __dmul_rn(__dsub_rn(u, g0), inv_eta)
              : __ddiv_rn(__dsub_rn(u, g0), eta);
}

// Outer recurrence — P/src/cheb.cpp:91,99-100.
__device__ __forceinline__ double outer(bool first, double g1, double g2,
                                        double fb, const StageArgs& a) {
  if (first) return __dadd_rn(g1, __dmul_rn(a.mudt, fb));
  return __dadd_rn(__dadd_rn(__dmul_rn(a.nu, g1), __dmul_rn(a.kappa, g2)),
                   __dmul_rn(a.mudt, fb));
}

__device__ __forceinline__ bool block_skip(const unsigned long long* ev,
                                           unsigned long long floor) {
  __shared__ int skip;
  if (threadIdx.x == 0 && threadIdx.y == 0)
    skip = (*(volatile const unsigned long long*)ev) < floor;
  __syncthreads();
  return skip != 0;
}

__device__ __forceinline__ void raise_if(unsigned long long* ev, bool bad,
                                         unsigned long long code) {
  if (bad) atomicMin(ev, code);
}

// Block min/max of ordered gate values, one atomic per block.
__device__ __forceinline__ void gate_range_block(unsigned long long* slot,
                                                 unsigned long long lo,
                                                 unsigned long long hi) {
  __shared__ unsigned long long slo[kThreads / 32], shi[kThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const int lane = threadIdx.x & 31;
  const int warp = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
  if (lane == 0) {
    slo[warp] = lo;
    shi[warp] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    const int nw = (blockDim.x * blockDim.y) >> 5;
    for (int w = 1; w < nw; ++w) {
      lo = min(lo, slo[w]);
      hi = max(hi, shi[w]);
    }
    lo = min(lo, slo[0]);
    hi = max(hi, shi[0]);
    if (lo != ~0ull) atomicMin(slot, lo);
    if (hi != 0ull) atomicMax(slot + 1, hi);
  }
}

// Epilogue shared by the stage-final kernels: store g_j, halo puts, finite
// check, and on the last stage the norm guard and gate range.
template <int DIM>
__device__ __forceinline__ void finish(const Geom& g, const Halo& h,
                                       const StageArgs& a, const Node<DIM>& n,
                                       const double o[4]) {
  bool bad = false;
  unsigned long long lo = ~0ull, hi = 0ull;
  if (n.valid) {
    const long long nn = g.nn;
    a.out[n.i] = o[0];
    a.out[nn + n.i] = o[1];
    a.out[2 * nn + n.i] = o[2];
    a.out[3 * nn + n.i] = o[3];
    if (h.put_lo && n.cz == 0) h.put_lo[n.ip] = o[0];
    if (h.put_hi && n.cz == g.nzl - 1) h.put_hi[n.ip] = o[0];
    bad = !(finite(o[0]) && finite(o[1]) && finite(o[2]) && finite(o[3]));
    if (a.last) {
      // ||V||_inf > 1e6 norm guard — P/src/simulate.cpp:222-227
      raise_if(a.event, fabs(o[0]) > 1e6,
               a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
      lo = min(ord_of(o[1]), min(ord_of(o[2]), ord_of(o[3])));
      hi = max(ord_of(o[1]), max(ord_of(o[2]), ord_of(o[3])));
    }
  }
  raise_if(a.event, bad,
           a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1) + a.m + 1));
  if (a.last) gate_range_block(a.gate_slot, lo, hi);
}

// ---------------------------------------------------------------------------
// K1: whole outer stage when m == 1 (the BASELINE configs' common case).
// One HBM pass: reads g_{j-1} (+ g_{j-2}), writes g_j.
// ---------------------------------------------------------------------------
template <int DIM, int FAST, int FIRST>
__global__ void __launch_bounds__(kThreads)
    k_stage_m1(const Geom g, const Halo h, const StageArgs a) {
  if (block_skip(a.event, level_floor(a.code_base, a.j, a.m, 1))) return;
  const Node<DIM> n = node_here<DIM>(g);
  const long long nn = g.nn;
  double o[4] = {0.0, 0.0, 0.0, 0.0};
  bool bad_in = false;
  if (n.valid) {
    const double* __restrict__ G = a.g1;
    const double V = __ldg(G + n.i);
    const double z[3] = {__ldg(G + nn + n.i), __ldg(G + 2 * nn + n.i),
                         __ldg(G + 3 * nn + n.i)};
    double lam[3], zinf[3];
    gate_coeffs<FAST>(V, lam, zinf);
    double ye[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) ye[k] = exp_euler(z[k], a.eta, lam[k], zinf[k]);
    const double fs =
        slow_v<FAST>(g, in_stim<DIM>(g, n) ? a.stim : 0.0, V, ye[0], ye[1], ye[2]);
    const double D = lap<DIM>(
        g, n, V, Ld{G}, [&](long long ip) { return __ldg(h.lo + ip); },
        [&](long long ip) { return __ldg(h.hi + ip); });
    const double mue = a.in_mueta[1];
    // inner stage 1: u_1 = y_E + mu'_1 eta (f_F(y_E) + fs); gate rows have
    // f_F = fs = 0 (P/src/monodomain.cpp:209-211,216-217)
    const double u[4] = {__dadd_rn(V, __dmul_rn(mue, __dadd_rn(D, fs))),
                         __dadd_rn(ye[0], __dmul_rn(mue, 0.0)),
                         __dadd_rn(ye[1], __dmul_rn(mue, 0.0)),
                         __dadd_rn(ye[2], __dmul_rn(mue, 0.0))};
    bad_in = !(finite(u[0]) && finite(u[1]) && finite(u[2]) && finite(u[3]));
    const double inv_eta = a.inv_eta;
    const double gv[4] = {V, z[0], z[1], z[2]};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double fb = avg_force<FAST>(u[k], gv[k], a.eta, inv_eta);
      const double g2 = FIRST ? 0.0 : __ldg(a.g2 + k * nn + n.i);
      o[k] = outer(FIRST, gv[k], g2, fb, a);
    }
  }
  raise_if(a.event, bad_in, a.code_base + (unsigned long long)((a.j - 1) * 2 + 1));
  finish<DIM>(g, h, a, n, o);
}

// ---------------------------------------------------------------------------
// m >= 2, first kernel of an outer stage: y_E, the frozen slow term and the
// first inner stage. Writes u_1 (V), fs (V) and y_E (gates).
// ---------------------------------------------------------------------------
template <int DIM, int FAST>
__global__ void __launch_bounds__(kThreads)
    k_stage_first(const Geom g, const Halo h, const StageArgs a) {
  if (block_skip(a.event, level_floor(a.code_base, a.j, a.m, 1))) return;
  const Node<DIM> n = node_here<DIM>(g);
  const long long nn = g.nn;
  bool bad = false;
  if (n.valid) {
    const double* __restrict__ G = a.g1;
    const double V = __ldg(G + n.i);
    const double z[3] = {__ldg(G + nn + n.i), __ldg(G + 2 * nn + n.i),
                         __ldg(G + 3 * nn + n.i)};
    double lam[3], zinf[3];
    gate_coeffs<FAST>(V, lam, zinf);
    double ye[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) ye[k] = exp_euler(z[k], a.eta, lam[k], zinf[k]);
    const double fs =
        slow_v<FAST>(g, in_stim<DIM>(g, n) ? a.stim : 0.0, V, ye[0], ye[1], ye[2]);
    const double D = lap<DIM>(
        g, n, V, Ld{G}, [&](long long ip) { return __ldg(h.lo + ip); },
        [&](long long ip) { return __ldg(h.hi + ip); });
    const double mue = a.in_mueta[1];
    const double u1 = __dadd_rn(V, __dmul_rn(mue, __dadd_rn(D, fs)));
    a.u[0][n.i] = u1;
    a.fs[n.i] = fs;
    a.ye[n.i] = ye[0];
    a.ye[nn + n.i] = ye[1];
    a.ye[2 * nn + n.i] = ye[2];
    if (h.put_lo && n.cz == 0) h.put_lo[n.ip] = u1;
    if (h.put_hi && n.cz == g.nzl - 1) h.put_hi[n.ip] = u1;
    bad = !(finite(u1) && finite(ye[0]) && finite(ye[1]) && finite(ye[2]));
  }
  raise_if(a.event, bad, a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1) + 1));
}

// ---------------------------------------------------------------------------
// m >= 2, inner stage k (2..m): u_k = nu'u_{k-1} + kappa'u_{k-2}
//   + mu'eta (f_F(u_{k-1}) + fs). The last one (k == m) also forms the
// averaged force, the outer recurrence and the epilogue.
// ---------------------------------------------------------------------------
template <int DIM, int FAST, int LASTK, int FIRST>
__global__ void __launch_bounds__(kThreads)
    k_stage_inner(const Geom g, const Halo h, const StageArgs a, const int k) {
  if (block_skip(a.event, level_floor(a.code_base, a.j, a.m, k))) return;
  const Node<DIM> n = node_here<DIM>(g);
  const long long nn = g.nn;
  bool bad = false;
  double o[4] = {0.0, 0.0, 0.0, 0.0};
  const double* __restrict__ um1 = a.u[(k - 2) % 3];
  const double* __restrict__ um2 = (k == 2) ? a.g1 : a.u[(k - 3) % 3];
  if (n.valid) {
    const double v1 = __ldg(um1 + n.i);
    const double v2 = __ldg(um2 + n.i);
    const double fs = __ldg(a.fs + n.i);
    const double D = lap<DIM>(
        g, n, v1, Ld{um1}, [&](long long ip) { return __ldg(h.lo + ip); },
        [&](long long ip) { return __ldg(h.hi + ip); });
    const double uk = __dadd_rn(
        __dadd_rn(__dmul_rn(a.in_nu[k], v1), __dmul_rn(a.in_kappa[k], v2)),
        __dmul_rn(a.in_mueta[k], __dadd_rn(D, fs)));
    bad = !finite(uk);
    if (!LASTK) {
      a.u[(k - 1) % 3][n.i] = uk;
      if (h.put_lo && n.cz == 0) h.put_lo[n.ip] = uk;
      if (h.put_hi && n.cz == g.nzl - 1) h.put_hi[n.ip] = uk;
    } else {
      // Gate rows of the inner iteration: u_1 = y_E + mu'_1 eta*0,
      // u_k = nu' u_{k-1} + kappa' u_{k-2} + mu'_k eta*0 (P/src/cheb.cpp:91,99)
      const double* __restrict__ G = a.g1;
      const double inv_eta = a.inv_eta;
      const double gv0 = __ldg(G + n.i);
      o[0] = outer(FIRST, gv0, FIRST ? 0.0 : __ldg(a.g2 + n.i),
                   avg_force<FAST>(uk, gv0, a.eta, inv_eta), a);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const double ye = __ldg(a.ye + q * nn + n.i);
        double p2 = ye;
        double p1 = __dadd_rn(ye, __dmul_rn(a.in_mueta[1], 0.0));
        for (int kk = 2; kk <= a.m; ++kk) {
          const double t = __dadd_rn(
              __dadd_rn(__dmul_rn(a.in_nu[kk], p1), __dmul_rn(a.in_kappa[kk], p2)),
              __dmul_rn(a.in_mueta[kk], 0.0));
          p2 = p1;
          p1 = t;
        }
        const double gq = __ldg(G + (q + 1) * nn + n.i);
        o[q + 1] = outer(FIRST, gq, FIRST ? 0.0 : __ldg(a.g2 + (q + 1) * nn + n.i),
                         avg_force<FAST>(p1, gq, a.eta, inv_eta), a);
      }
    }
  }
  raise_if(a.event, bad,
           a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1) + k));
  if (LASTK) finish<DIM>(g, h, a, n, o);
}

// ---------------------------------------------------------------------------
// Operator evaluations (f_F, f_S, exp_part) and the power iteration.
// ---------------------------------------------------------------------------
template <int DIM>
__global__ void __launch_bounds__(kThreads)
    k_rhs(const Geom g, const Halo h, int which, const double* __restrict__ y,
          double stim, double* __restrict__ out) {
  const Node<DIM> n = node_here<DIM>(g);
  if (!n.valid) return;
  const long long nn = g.nn;
  const double V = y[n.i];
  double r;
  if ((which & 15) == 0) {
    r = lap<DIM>(g, n, V, Ld{y}, [&](long long ip) { return h.lo[ip]; },
                 [&](long long ip) { return h.hi[ip]; });
  } else {
    r = slow_v<0>(g, in_stim<DIM>(g, n) ? stim : 0.0, V, y[nn + n.i],
                  y[2 * nn + n.i], y[3 * nn + n.i]);
  }
  out[n.i] = r;
  // gate rows of the mRKC split (which bits 4..6): Lambda_g (z_g - z_inf_g)
  // (gate_rows, P/src/monodomain.cpp:223-236)
  const int gm = (which >> 4) & 7;
  double l[3] = {0.0, 0.0, 0.0}, zi[3] = {0.0, 0.0, 0.0};
  if (gm) hh_gate_coeffs_ref(V, l, zi);
#pragma unroll
  for (int q = 0; q < 3; ++q)
    out[(q + 1) * nn + n.i] =
        (gm >> q & 1) ? __dmul_rn(l[q], __dsub_rn(y[(q + 1) * nn + n.i], zi[q])) : 0.0;
  // aux rows (EMRKC_MODEL_HH_AUX): f_F 0, f_S aux_rates_field
  // (P/src/monodomain.cpp:191-205, 214-221)
  for (int a = 0; a < g.naux; ++a) {
    const long long k = (4 + a) * nn + n.i;
    out[k] = (which & 15) == 0 ? 0.0 : aux_rate_ref(a, V, y[k]);
  }
}

// mRKC inner stage k of outer stage j, reference operation order
// (rkc_iteration, P/src/cheb.cpp:84-105; averaged_force_mrkc,
// P/src/multirate.cpp:60-76): f_u = f_F_with_gates(u) + fs with the slow
// term fs = f_S_with_gates(g_{j-1}) frozen at k == 1; at k == m the averaged
// force (u_m - g_{j-1}) / eta enters the outer recurrence.
template <int DIM>
__global__ void __launch_bounds__(kThreads)
    k_mrkc_stage(const Geom g, const MrkcArgs a) {
  const Node<DIM> n = node_here<DIM>(g);
  if (!n.valid) return;
  if (*(volatile const unsigned long long*)a.event < level_floor(a.code_base, a.j, a.m, a.k)) return;  // aborted earlier
  const long long nn = g.nn, i = n.i;
  const double* U = a.um1;
  const double V = U[i];
  const auto none = [](long long) { return 0.0; };  // whole grid: no ghost planes
  double f[4];
  f[0] = lap<DIM>(g, n, V, Ld{U}, none, none);
  double l[3], zi[3];
  hh_gate_coeffs_ref(V, l, zi);
#pragma unroll
  for (int q = 0; q < 3; ++q)
    f[q + 1] = (a.stiff >> q & 1) ? __dmul_rn(l[q], __dsub_rn(U[(q + 1) * nn + i], zi[q])) : 0.0;
  double fs[4];
  if (a.k == 1) {  // U == g_{j-1}
    fs[0] = slow_v<0>(g, in_stim<DIM>(g, n) ? a.stim : 0.0, V, U[nn + i], U[2 * nn + i],
                      U[3 * nn + i]);
#pragma unroll
    for (int q = 0; q < 3; ++q)
      fs[q + 1] = (a.stiff >> q & 1) ? 0.0
                                     : __dmul_rn(l[q], __dsub_rn(U[(q + 1) * nn + i], zi[q]));
    if (a.m > 1)
#pragma unroll
      for (int c = 0; c < 4; ++c) a.fs[c * nn + i] = fs[c];
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) fs[c] = a.fs[c * nn + i];
  }
  double u[4];
  bool bad = false;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double fc = __dadd_rn(f[c], fs[c]);
    const long long jc = c * nn + i;
    u[c] = a.k == 1 ? __dadd_rn(U[jc], __dmul_rn(a.mueta, fc))
                    : __dadd_rn(__dadd_rn(__dmul_rn(a.nu, U[jc]), __dmul_rn(a.kappa, a.um2[jc])),
                                __dmul_rn(a.mueta, fc));
    bad |= !isfinite(u[c]);
  }
  const unsigned long long base = a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1));
  if (bad) atomicMin(a.event, base + a.k);
  if (a.k < a.m) {
#pragma unroll
    for (int c = 0; c < 4; ++c) a.uk[c * nn + i] = u[c];
    return;
  }
  bool bad_out = false;
  double o[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const long long jc = c * nn + i;
    const double y = a.g1[jc];
    const double force = __ddiv_rn(__dsub_rn(u[c], y), a.eta);  // multirate.cpp:74
    o[c] = a.j == 1 ? __dadd_rn(y, __dmul_rn(a.mudt, force))
                    : __dadd_rn(__dadd_rn(__dmul_rn(a.onu, y), __dmul_rn(a.okappa, a.g2[jc])),
                                __dmul_rn(a.mudt, force));
    a.out[jc] = o[c];
    bad_out |= !isfinite(o[c]);
  }
  if (bad_out) atomicMin(a.event, base + a.m + 1);
  if (a.last && !(fabs(o[0]) <= 1e6))
    atomicMin(a.event, a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
}

template <int DIM>
__global__ void __launch_bounds__(kThreads)
    k_exp_part(const Geom g, const double* __restrict__ y,
               double* __restrict__ lam, double* __restrict__ yinf) {
  const Node<DIM> n = node_here<DIM>(g);
  if (!n.valid) return;
  const long long nn = g.nn;
  double l[3], zi[3];
  hh_gate_coeffs_ref(y[n.i], l, zi);
  lam[n.i] = 0.0;
  yinf[n.i] = 0.0;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    lam[(q + 1) * nn + n.i] = l[q];
    yinf[(q + 1) * nn + n.i] = zi[q];
  }
  for (int a = 0; a < g.naux; ++a) {  // exp_part is zero on the aux rows
    lam[(4 + a) * nn + n.i] = 0.0;
    yinf[(4 + a) * nn + n.i] = 0.0;
  }
}

constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double x) {
  __shared__ double sh[kRedThreads / 32];
  for (int o = 16; o > 0; o >>= 1) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = x;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kRedThreads / 32; ++w) t = __dadd_rn(t, sh[w]);
  return t;  // valid in thread 0
}

// vout = f(y + q v) - f(y) with partial sums of vout^2 (fixed grid =>
// deterministic), P/src/spectral.cpp:52-56.
template <int DIM>
__global__ void __launch_bounds__(kRedThreads)
    k_power(const Geom g, int which, const double* __restrict__ y,
            const double* __restrict__ v, const double q,
            const double* __restrict__ fy, double stim,
            double* __restrict__ vout, const double* gy_lo,
            const double* gy_hi, const double* gv_lo, const double* gv_hi,
            double* __restrict__ partial) {
  const long long nn = g.nn;
  double acc = 0.0;
  const LdZ z{y, v, q};
  for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < nn;
       i += (long long)gridDim.x * kRedThreads) {
    const Node<DIM> n = node_flat<DIM>(g, i);
    const double zv = z(i);
    double fz;
    if ((which & 15) == 0) {
      fz = lap<DIM>(
          g, n, zv, z,
          [&](long long ip) { return __dadd_rn(gy_lo[ip], __dmul_rn(q, gv_lo[ip])); },
          [&](long long ip) { return __dadd_rn(gy_hi[ip], __dmul_rn(q, gv_hi[ip])); });
    } else {
      fz = slow_v<0>(g, in_stim<DIM>(g, n) ? stim : 0.0, zv, z(nn + i),
                     z(2 * nn + i), z(3 * nn + i));
    }
    const double d = __dsub_rn(fz, fy[i]);
    vout[i] = d;
    acc = __dadd_rn(acc, __dmul_rn(d, d));
    const int gm = (which >> 4) & 7;  // gate rows of the mRKC split
    double l[3] = {0.0, 0.0, 0.0}, zi[3] = {0.0, 0.0, 0.0};
    if (gm) hh_gate_coeffs_ref(zv, l, zi);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double dq = 0.0;
      if (gm >> q & 1) {
        const long long k = (q + 1) * nn + i;
        dq = __dsub_rn(__dmul_rn(l[q], __dsub_rn(z(k), zi[q])), fy[k]);
        acc = __dadd_rn(acc, __dmul_rn(dq, dq));
      }
      vout[(q + 1) * nn + i] = dq;
    }
    // aux rows: f_S(z) - f_S(y) (f_F is zero there)
    for (int a = 0; a < g.naux; ++a) {
      const long long k = (4 + a) * nn + i;
      double da = 0.0;
      if ((which & 15) != 0) {
        da = __dsub_rn(aux_rate_ref(a, zv, z(k)), fy[k]);
        acc = __dadd_rn(acc, __dmul_rn(da, da));
      }
      vout[k] = da;
    }
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kRedThreads)
    k_norm2_partial(const double* __restrict__ x, long long len,
                    double* __restrict__ partial) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < len;
       i += (long long)gridDim.x * kRedThreads)
    acc = __dadd_rn(acc, __dmul_rn(x[i], x[i]));
  const double t = block_sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// Trapezoid-weighted sums of (a - b)^2 and b^2 over one node field
// (rel_l2_error / l2_norm / quadrature_weights, P/src/monodomain.cpp:52-63,
// 88-110): weight 1/2 per axis where the node sits on that axis' boundary.
__global__ void __launch_bounds__(kRedThreads)
    k_rel_l2_partial(const Geom g, const double* __restrict__ a, const double* __restrict__ b,
                     double* __restrict__ partial) {
  double sd = 0.0, sb = 0.0;
  const long long nn = g.nn;
  for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < nn;
       i += (long long)gridDim.x * kRedThreads) {
    double w = 1.0;
    long long r = i;
    const long long na[3] = {g.n0, g.n1, g.nzl};
    for (int ax = 0; ax < g.dim; ++ax) {
      const long long ia = r % na[ax];
      r /= na[ax];
      if (ia == 0 || ia == na[ax] - 1) w *= 0.5;
    }
    const double d = a[i] - b[i];
    sd = __dadd_rn(sd, w * d * d);
    sb = __dadd_rn(sb, w * b[i] * b[i]);
  }
  const double td = block_sum(sd);
  __syncthreads();
  const double tb = block_sum(sb);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = td;
    partial[2 * blockIdx.x + 1] = tb;
  }
}

__global__ void __launch_bounds__(kRedThreads)
    k_sum_partials2(const double* __restrict__ partial, int n, double* __restrict__ out) {
  double a0 = 0.0, a1 = 0.0;
  for (int i = threadIdx.x; i < n; i += kRedThreads) {
    a0 = __dadd_rn(a0, partial[2 * i]);
    a1 = __dadd_rn(a1, partial[2 * i + 1]);
  }
  const double t0 = block_sum(a0);
  __syncthreads();
  const double t1 = block_sum(a1);
  if (threadIdx.x == 0) {
    out[0] = t0;
    out[1] = t1;
  }
}

// ---- IMEX-RL (P/src/baselines.cpp:89-190) ---------------------------------
// sqrt of the trapezoid node weight (quadrature_weights,
// P/src/monodomain.cpp:52-63): 1/2 per axis on which the node is a boundary.
template <int DIM>
__device__ __forceinline__ double sqrt_w(const Geom& g, long long i) {
  double w = 1.0;
  long long r = i;
  const long long na[3] = {g.n0, g.n1, g.nzl};
#pragma unroll
  for (int ax = 0; ax < DIM; ++ax) {
    const long long ia = r % na[ax];
    r /= na[ax];
    if (ia == 0 || ia == na[ax] - 1) w *= 0.5;
  }
  return sqrt(w);
}

// Rush-Larsen part (rush_larsen_update, baselines.cpp:89-128) and the CG
// right-hand side / warm start (:164-168): gates of `out`, b, x; partials
// of ||b||^2.
template <int DIM>
__global__ void __launch_bounds__(kRedThreads)
    k_imex_prep(const Geom g, const double* __restrict__ y, double dt, double stim,
                double* __restrict__ out, double* __restrict__ b, double* __restrict__ x,
                double* __restrict__ partial) {
  const long long nn = g.nn;
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < nn;
       i += (long long)gridDim.x * kRedThreads) {
    const Node<DIM> n = node_flat<DIM>(g, i);
    const double V = y[i];
    double l[3], zi[3], zn[3];
    hh_gate_coeffs_ref(V, l, zi);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double z = y[(q + 1) * nn + i];
      zn[q] = __dadd_rn(z, __dmul_rn(expm1(__dmul_rn(dt, l[q])), __dsub_rn(z, zi[q])));
      out[(q + 1) * nn + i] = zn[q];
    }
    const double vr = slow_v<0>(g, in_stim<DIM>(g, n) ? stim : 0.0, V, zn[0], zn[1], zn[2]);
    const double sw = sqrt_w<DIM>(g, i);
    const double bi = __dmul_rn(sw, __dadd_rn(V, __dmul_rn(dt, vr)));
    b[i] = bi;
    x[i] = __dmul_rn(sw, V);
    acc = __dadd_rn(acc, __dmul_rn(bi, bi));
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// op(u) = u - dt sqrt(w) D(u / sqrt(w)) at node i (the CG operator, :154-158)
template <int DIM>
__device__ __forceinline__ double cg_op(const Geom& g, const Node<DIM>& n,
                                        const double* __restrict__ u, double dt) {
  const auto f = [&](long long j) { return __ddiv_rn(u[j], sqrt_w<DIM>(g, j)); };
  const auto none = [](long long) { return 0.0; };
  const double d = lap<DIM>(g, n, f(n.i), f, none, none);
  return __dsub_rn(u[n.i], __dmul_rn(__dmul_rn(dt, sqrt_w<DIM>(g, n.i)), d));
}

// r = b - op(x), z = r / diag (Jacobi, diag <= 0: none), p = z; partials
// of r.z and r.r (cg_solve, :41-49)
template <int DIM>
__global__ void __launch_bounds__(kRedThreads)
    k_cg_init(const Geom g, double dt, double diag, const double* __restrict__ b,
              const double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
              double* __restrict__ p, double* __restrict__ partial) {
  const long long nn = g.nn;
  double arz = 0.0, arr = 0.0;
  for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < nn;
       i += (long long)gridDim.x * kRedThreads) {
    const Node<DIM> n = node_flat<DIM>(g, i);
    const double ri = __dsub_rn(b[i], cg_op<DIM>(g, n, x, dt));
    const double zz = diag > 0.0 ? __ddiv_rn(ri, diag) : ri;
    r[i] = ri;
    z[i] = zz;
    p[i] = zz;
    arz = __dadd_rn(arz, __dmul_rn(ri, zz));
    arr = __dadd_rn(arr, __dmul_rn(ri, ri));
  }
  const double t0 = block_sum(arz);
  __syncthreads();
  const double t1 = block_sum(arr);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = t0;
    partial[2 * blockIdx.x + 1] = t1;
  }
}

// One-block scalar steps of cg_solve. phase 0: ||b|| and the initial r.z,
// r.r (loop entry); phase 1: alpha = rz / p.q; phase 2: beta, rnorm, the
// loop test (while rnorm > tol, iterations < max_iters).
__global__ void __launch_bounds__(kRedThreads)
    k_cg_scalar(const double* __restrict__ partial, int n, int phase, CgScalars* cs,
                const double* __restrict__ partial_b, double rel_tol, long long max_it) {
  double a0 = 0.0, a1 = 0.0, ab = 0.0;
  for (int i = threadIdx.x; i < n; i += kRedThreads) {
    if (phase == 1) {
      a0 = __dadd_rn(a0, partial[i]);
    } else {
      a0 = __dadd_rn(a0, partial[2 * i]);
      a1 = __dadd_rn(a1, partial[2 * i + 1]);
    }
    if (phase == 0) ab = __dadd_rn(ab, partial_b[i]);
  }
  const double t0 = block_sum(a0);
  __syncthreads();
  const double t1 = block_sum(a1);
  __syncthreads();
  const double tb = block_sum(ab);
  if (threadIdx.x != 0) return;
  if (phase == 0) {
    cs->nb2 = tb;
    cs->tol = rel_tol * sqrt(tb);
    cs->rz = t0;
    cs->rr = t1;
    cs->it = 0;
    cs->max_it = max_it;
    cs->converged = 1;
    cs->done = !(sqrt(t1) > cs->tol);
    return;
  }
  if (cs->done) return;
  if (phase == 1) {
    cs->pq = t0;
    cs->alpha = __ddiv_rn(cs->rz, t0);
    return;
  }
  cs->beta = __ddiv_rn(t0, cs->rz);
  cs->rz = t0;
  cs->rr = t1;
  cs->it += 1;
  if (!(sqrt(t1) > cs->tol)) {
    cs->done = 1;
  } else if (cs->it >= cs->max_it) {
    cs->done = 1;
    cs->converged = 0;
  }
}

// q = op(p); partials of p.q
template <int DIM>
__global__ void __launch_bounds__(kRedThreads)
    k_cg_apply(const Geom g, double dt, const double* __restrict__ p, double* __restrict__ q,
               double* __restrict__ partial, const CgScalars* cs) {
  if (cs->done) return;
  const long long nn = g.nn;
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < nn;
       i += (long long)gridDim.x * kRedThreads) {
    const Node<DIM> n = node_flat<DIM>(g, i);
    const double qi = cg_op<DIM>(g, n, p, dt);
    q[i] = qi;
    acc = __dadd_rn(acc, __dmul_rn(p[i], qi));
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// x += alpha p, r -= alpha q, z = r / diag; partials of r.z, r.r
__global__ void __launch_bounds__(kRedThreads)
    k_cg_update(long long nn, double diag, double* __restrict__ x, double* __restrict__ r,
                double* __restrict__ z, const double* __restrict__ p,
                const double* __restrict__ q, double* __restrict__ partial,
                const CgScalars* cs) {
  if (cs->done) return;
  const double alpha = cs->alpha;
  double arz = 0.0, arr = 0.0;
  for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < nn;
       i += (long long)gridDim.x * kRedThreads) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    const double ri = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
    r[i] = ri;
    const double zz = diag > 0.0 ? __ddiv_rn(ri, diag) : ri;
    z[i] = zz;
    arz = __dadd_rn(arz, __dmul_rn(ri, zz));
    arr = __dadd_rn(arr, __dmul_rn(ri, ri));
  }
  const double t0 = block_sum(arz);
  __syncthreads();
  const double t1 = block_sum(arr);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = t0;
    partial[2 * blockIdx.x + 1] = t1;
  }
}

// p = z + beta p (after the loop test: skipped once done)
__global__ void __launch_bounds__(kRedThreads)
    k_cg_dir(long long nn, const double* __restrict__ z, double* __restrict__ p,
             const CgScalars* cs) {
  if (cs->done) return;
  const double beta = cs->beta;
  for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < nn;
       i += (long long)gridDim.x * kRedThreads)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

// V_new = x / sqrt(w) (:185); x = 0 when ||b|| = 0 (:25-29)
template <int DIM>
__global__ void __launch_bounds__(kRedThreads)
    k_cg_finish(const Geom g, const double* __restrict__ x, double* __restrict__ out,
                const CgScalars* cs) {
  const bool zero = cs->nb2 == 0.0;
  for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < g.nn;
       i += (long long)gridDim.x * kRedThreads)
    out[i] = zero ? 0.0 : __dmul_rn(__ddiv_rn(1.0, sqrt_w<DIM>(g, i)), x[i]);
}

__global__ void __launch_bounds__(kRedThreads)
    k_sum_partials(const double* __restrict__ partial, int n,
                   double* __restrict__ out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += kRedThreads) acc = __dadd_rn(acc, partial[i]);
  const double t = block_sum(acc);
  if (threadIdx.x == 0) *out = t;
}

template <int DIM>
__global__ void __launch_bounds__(kThreads)
    k_gate_range(const Geom g, const double* __restrict__ y,
                 unsigned long long* slot) {
  const Node<DIM> n = node_here<DIM>(g);
  unsigned long long lo = ~0ull, hi = 0ull;
  if (n.valid) {
    const long long nn = g.nn;
    for (int q = 1; q <= 3; ++q) {
      const double v = y[q * nn + n.i];
      if (v != v) continue;  // NaN never wins std::min / std::max (simulate.cpp:82-83)
      const unsigned long long o = ord_of(v);
      lo = min(lo, o);
      hi = max(hi, o);
    }
  }
  gate_range_block(slot, lo, hi);
}

// min over the abort words of all slabs of a group into this slab's word
// (pointers passed by value: up to 16 slabs)
__global__ void k_fold_events_arr(
    unsigned long long* dst, unsigned long long* s0, unsigned long long* s1,
    unsigned long long* s2, unsigned long long* s3, unsigned long long* s4,
    unsigned long long* s5, unsigned long long* s6, unsigned long long* s7,
    unsigned long long* s8, unsigned long long* s9, unsigned long long* s10,
    unsigned long long* s11, unsigned long long* s12, unsigned long long* s13,
    unsigned long long* s14, unsigned long long* s15, int n) {
  unsigned long long* src[16] = {s0, s1, s2,  s3,  s4,  s5,  s6,  s7,
                                 s8, s9, s10, s11, s12, s13, s14, s15};
  unsigned long long m = *(volatile unsigned long long*)dst;
  for (int q = 0; q < n; ++q) m = min(m, *(volatile unsigned long long*)src[q]);
  *dst = m;
}

__global__ void k_fill_u64(unsigned long long* p, long long n,
                           unsigned long long v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

template <int DIM>
dim3 grid_of(const Geom& g) {
  if (DIM == 3) return dim3((g.n0 + BX - 1) / BX, (g.n1 + BY - 1) / BY, g.nzl);
  if (DIM == 2) return dim3((g.n0 + BX - 1) / BX, (g.nzl + BY - 1) / BY, 1);
  return dim3((g.nzl + BX * BY - 1) / (BX * BY), 1, 1);
}

}  // namespace

int power_blocks() { return 148 * 8; }

#define DISPATCH_DIM(g, ...)                                \
  switch ((g).dim) {                                        \
    case 1: { constexpr int D = 1; __VA_ARGS__; break; }    \
    case 2: { constexpr int D = 2; __VA_ARGS__; break; }    \
    default: { constexpr int D = 3; __VA_ARGS__; break; }   \
  }

cudaError_t launch_stage_m1(const Geom& g, const Halo& h, const StageArgs& a,
                            int fast, cudaStream_t st) {
  const dim3 blk(BX, BY);
  const bool first = a.j == 1;
  DISPATCH_DIM(g, {
    const dim3 grd = grid_of<D>(g);
    if (fast) {
      if (first) k_stage_m1<D, 1, 1><<<grd, blk, 0, st>>>(g, h, a);
      else k_stage_m1<D, 1, 0><<<grd, blk, 0, st>>>(g, h, a);
    } else {
      if (first) k_stage_m1<D, 0, 1><<<grd, blk, 0, st>>>(g, h, a);
      else k_stage_m1<D, 0, 0><<<grd, blk, 0, st>>>(g, h, a);
    }
  });
  return cudaGetLastError();
}

cudaError_t launch_stage_first(const Geom& g, const Halo& h,
                               const StageArgs& a, int fast, cudaStream_t st) {
  const dim3 blk(BX, BY);
  DISPATCH_DIM(g, {
    const dim3 grd = grid_of<D>(g);
    if (fast) k_stage_first<D, 1><<<grd, blk, 0, st>>>(g, h, a);
    else k_stage_first<D, 0><<<grd, blk, 0, st>>>(g, h, a);
  });
  return cudaGetLastError();
}

cudaError_t launch_stage_inner(const Geom& g, const Halo& h,
                               const StageArgs& a, int k, int fast,
                               cudaStream_t st) {
  const dim3 blk(BX, BY);
  const bool lastk = k == a.m;
  const bool first = a.j == 1;
  DISPATCH_DIM(g, {
    const dim3 grd = grid_of<D>(g);
    if (!lastk) k_stage_inner<D, 1, 0, 0><<<grd, blk, 0, st>>>(g, h, a, k);
    else if (fast && first) k_stage_inner<D, 1, 1, 1><<<grd, blk, 0, st>>>(g, h, a, k);
    else if (fast) k_stage_inner<D, 1, 1, 0><<<grd, blk, 0, st>>>(g, h, a, k);
    else if (first) k_stage_inner<D, 0, 1, 1><<<grd, blk, 0, st>>>(g, h, a, k);
    else k_stage_inner<D, 0, 1, 0><<<grd, blk, 0, st>>>(g, h, a, k);
  });
  return cudaGetLastError();
}

cudaError_t launch_rhs(const Geom& g, const Halo& h, int which,
                       const double* y, double stim, double* out,
                       cudaStream_t st) {
  const dim3 blk(BX, BY);
  DISPATCH_DIM(g, { k_rhs<D><<<grid_of<D>(g), blk, 0, st>>>(g, h, which, y, stim, out); });
  return cudaGetLastError();
}

cudaError_t launch_mrkc_stage(const Geom& g, const MrkcArgs& a, cudaStream_t st) {
  const dim3 blk(BX, BY);
  DISPATCH_DIM(g, { k_mrkc_stage<D><<<grid_of<D>(g), blk, 0, st>>>(g, a); });
  return cudaGetLastError();
}

cudaError_t launch_imex_prep(const Geom& g, const double* y, double dt, double stim,
                             double* out, double* b, double* x, double* partial, int nblocks,
                             cudaStream_t st) {
  DISPATCH_DIM(g, {
    k_imex_prep<D><<<nblocks, kRedThreads, 0, st>>>(g, y, dt, stim, out, b, x, partial);
  });
  return cudaGetLastError();
}

cudaError_t launch_cg_init(const Geom& g, double dt, double diag, const double* b,
                           const double* x, double* r, double* z, double* p, double* partial,
                           int nblocks, CgScalars* cs, double rel_tol, long long max_it,
                           const double* partial_b, cudaStream_t st) {
  DISPATCH_DIM(g, {
    k_cg_init<D><<<nblocks, kRedThreads, 0, st>>>(g, dt, diag, b, x, r, z, p, partial);
  });
  k_cg_scalar<<<1, kRedThreads, 0, st>>>(partial, nblocks, 0, cs, partial_b, rel_tol, max_it);
  return cudaGetLastError();
}

cudaError_t launch_cg_iter(const Geom& g, double dt, double diag, double* x, double* r,
                           double* z, double* p, double* q, double* partial, int nblocks,
                           CgScalars* cs, cudaStream_t st) {
  DISPATCH_DIM(g, {
    k_cg_apply<D><<<nblocks, kRedThreads, 0, st>>>(g, dt, p, q, partial, cs);
  });
  k_cg_scalar<<<1, kRedThreads, 0, st>>>(partial, nblocks, 1, cs, nullptr, 0.0, 0);
  k_cg_update<<<nblocks, kRedThreads, 0, st>>>(g.nn, diag, x, r, z, p, q, partial, cs);
  k_cg_scalar<<<1, kRedThreads, 0, st>>>(partial, nblocks, 2, cs, nullptr, 0.0, 0);
  k_cg_dir<<<nblocks, kRedThreads, 0, st>>>(g.nn, z, p, cs);
  return cudaGetLastError();
}

cudaError_t launch_cg_finish(const Geom& g, const double* x, double* out, const CgScalars* cs,
                             cudaStream_t st) {
  DISPATCH_DIM(g, { k_cg_finish<D><<<power_blocks(), kRedThreads, 0, st>>>(g, x, out, cs); });
  return cudaGetLastError();
}

// norm guard of run_simulation (max_abs_v > 1e6, non-finite -> inf;
// P/src/simulate.cpp:67-74,222-227): flag = 1 if any |V| > 1e6 or NaN
__global__ void k_v_guard(long long nn, const double* __restrict__ y, int* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nn;
       i += (long long)gridDim.x * blockDim.x)
    if (!(fabs(y[i]) <= 1e6)) atomicOr(flag, 1);
}

cudaError_t launch_v_guard(long long nn, const double* y, int* flag, cudaStream_t st) {
  k_v_guard<<<power_blocks(), 256, 0, st>>>(nn, y, flag);
  return cudaGetLastError();
}

double diffusion_diag(const Geom& g) {
  // diffusion_apply(e_0)[0]: node 0 is a corner; the mirror doubles the
  // neighbour weight of every axis, the centre term is -2 w_a per axis
  // (P/src/monodomain.cpp:73-90) -> sum over axes of w_a (0 - 2 + 0)
  double d = 0.0;
  for (int a = 0; a < g.dim; ++a) d += g.w[a] * (0.0 - 2.0 * 1.0 + 0.0);
  return d;
}

cudaError_t launch_exp_part(const Geom& g, const double* y, double* lam,
                            double* yinf, cudaStream_t st) {
  const dim3 blk(BX, BY);
  DISPATCH_DIM(g, { k_exp_part<D><<<grid_of<D>(g), blk, 0, st>>>(g, y, lam, yinf); });
  return cudaGetLastError();
}

cudaError_t launch_power(const Geom& g, int which, const double* y,
                         const double* v, double q,
                         const double* fy, double stim, double* vout,
                         const double* gy_lo, const double* gy_hi,
                         const double* gv_lo, const double* gv_hi,
                         double* partial, int nblocks, cudaStream_t st) {
  DISPATCH_DIM(g, {
    k_power<D><<<nblocks, kRedThreads, 0, st>>>(g, which, y, v, q, fy, stim,
                                                vout, gy_lo, gy_hi, gv_lo, gv_hi,
                                                partial);
  });
  return cudaGetLastError();
}

// Sum of squares in the reference's SERIAL order (P/src/spectral.cpp:10-14:
// s += x * x, i = 0 .. n-1, no FMA), continuing from acc: one block, the
// squares staged through a double-buffered shared chunk by warps 1..7 while
// thread 0 runs the dependent add chain. Bit-identical to the reference's
// norm2 (so the power iteration's q = delta / ||v|| and every z = y + q v
// are too); a run of segments chained through acc covers a vector held in
// several pieces (SoA blocks of z-slabs, in global order).
constexpr int kSerT = 256, kSerC = 2048;
__global__ void __launch_bounds__(kSerT) k_sumsq_serial(const double* __restrict__ x, long long n,
                                                        double acc, double* out) {
  __shared__ double buf[2][kSerC];
  const int t = threadIdx.x;
  const long long nch = (n + kSerC - 1) / kSerC;
  for (int k = t; k < kSerC; k += kSerT) buf[0][k] = k < n ? __dmul_rn(x[k], x[k]) : 0.0;
  __syncthreads();
  double s = acc;
  for (long long c = 0; c < nch; ++c) {
    const int cur = (int)(c & 1);
    if (t >= 32) {
      if (c + 1 < nch) {
        const long long base = (c + 1) * kSerC;
        for (int k = t - 32; k < kSerC; k += kSerT - 32) {
          const long long i = base + k;
          buf[cur ^ 1][k] = i < n ? __dmul_rn(x[i], x[i]) : 0.0;
        }
      }
    } else if (t == 0) {
      const int len = (int)min((long long)kSerC, n - c * kSerC);
      const double* b = buf[cur];
      int k = 0;
      for (; k + 8 <= len; k += 8) {
        const double b0 = b[k], b1 = b[k + 1], b2 = b[k + 2], b3 = b[k + 3];
        const double b4 = b[k + 4], b5 = b[k + 5], b6 = b[k + 6], b7 = b[k + 7];
        s = __dadd_rn(s, b0);
        s = __dadd_rn(s, b1);
        s = __dadd_rn(s, b2);
        s = __dadd_rn(s, b3);
        s = __dadd_rn(s, b4);
        s = __dadd_rn(s, b5);
        s = __dadd_rn(s, b6);
        s = __dadd_rn(s, b7);
      }
      for (; k < len; ++k) s = __dadd_rn(s, b[k]);
    }
    __syncthreads();
  }
  if (t == 0) *out = s;
}

cudaError_t launch_sumsq_serial(const double* x, long long len, double acc, double* out,
                                cudaStream_t st) {
  k_sumsq_serial<<<1, kSerT, 0, st>>>(x, len, acc, out);
  return cudaGetLastError();
}

cudaError_t launch_norm2_partial(const double* x, long long len,
                                 double* partial, int nblocks,
                                 cudaStream_t st) {
  k_norm2_partial<<<nblocks, kRedThreads, 0, st>>>(x, len, partial);
  return cudaGetLastError();
}

cudaError_t launch_rel_l2(const Geom& g, const double* a, const double* b, double* partial,
                          int nblocks, double* out2, cudaStream_t st) {
  k_rel_l2_partial<<<nblocks, kRedThreads, 0, st>>>(g, a, b, partial);
  k_sum_partials2<<<1, kRedThreads, 0, st>>>(partial, nblocks, out2);
  return cudaGetLastError();
}

cudaError_t launch_sum_partials(const double* partial, int nblocks,
                                double* out, cudaStream_t st) {
  k_sum_partials<<<1, kRedThreads, 0, st>>>(partial, nblocks, out);
  return cudaGetLastError();
}

cudaError_t launch_gate_range(const Geom& g, const double* y,
                              unsigned long long* slot, cudaStream_t st) {
  const dim3 blk(BX, BY);
  DISPATCH_DIM(g, { k_gate_range<D><<<grid_of<D>(g), blk, 0, st>>>(g, y, slot); });
  return cudaGetLastError();
}

cudaError_t launch_fold_events(unsigned long long* dst,
                               unsigned long long* const* src, int n,
                               cudaStream_t st) {
  if (n > 16) return cudaErrorInvalidValue;
  struct P { unsigned long long* p[16]; } arr{};
  for (int q = 0; q < n; ++q) arr.p[q] = src[q];
  k_fold_events_arr<<<1, 1, 0, st>>>(dst, arr.p[0], arr.p[1], arr.p[2], arr.p[3], arr.p[4],
                                     arr.p[5], arr.p[6], arr.p[7], arr.p[8], arr.p[9],
                                     arr.p[10], arr.p[11], arr.p[12], arr.p[13], arr.p[14],
                                     arr.p[15], n);
  return cudaGetLastError();
}

cudaError_t launch_fill_u64(unsigned long long* p, long long n,
                            unsigned long long v, cudaStream_t st) {
  const int blocks = (int)((n + 255) / 256 > 1024 ? 1024 : (n + 255) / 256);
  k_fill_u64<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(p, n, v);
  return cudaGetLastError();
}

}  // namespace emrkc_k
