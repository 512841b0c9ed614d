// kernels_fast.cu — the default (fast) emRKC kernels for sm_100a.
//
// Same step as kernels.cu with the per-node arithmetic cut to
// what the FP64 pipe can sustain at HBM speed:
//  * z-marching (2.5-D): each thread owns one (x, y) column and walks `zc`
//    consecutive planes of its slab, keeping V(z-1), V(z), V(z+1) in
//    registers; x/y neighbours come from L1. Block prologue (abort-word
//    check, 2 KiB exp table) and epilogue (gate range, norm guard) are
//    amortised over the column.
//  * ionic model through fast_math.cuh (3 + 3 table exps, one reciprocal).
//  * recurrences in FMA form, and the algebra of SURVEY §8(a): f_F and f_S
//    vanish on gate rows, so a gate's inner iterate is y_E (nu' + kappa' = 1)
//    and its outer update is base + (mu_j dt / eta) (y_E - z); only V needs
//    the stencil recurrence.
// All of this moves results by rounding only; tests/test_gpu_parity.py holds
// the default path to the reference within rel-L2 1e-9 (north_star).
//
// Kernels:
//  k_m1_fast    m == 1: one HBM pass per outer stage (reads g_{j-1}[, g_{j-2}],
//               writes g_j): the BASELINE configs 1-3 case.
//  k_ion_fast   m >= 2, inner stage 1: ionic + gates of g_j (final), fs, u_1.
//  k_vin_fast   m >= 2, inner stage k >= 2, V block only; the k == m launch
//               forms V of g_j.
#include <cstdio>

#include "aux.cuh"
#include "fast_math.cuh"
#include "hh.cuh"
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include <cooperative_groups.h>

#include "kernels.h"
#include "tma.cuh"

#ifndef EMRKC_EXPERIMENTAL
#define EMRKC_EXPERIMENTAL 0
#endif

namespace emrkc_k {

using namespace emrkc_dev;

namespace {

constexpr int FBX = 32;
constexpr int FBY = 4;
constexpr int kFThreads = FBX * FBY;

template <int DIM>
struct Col {
  int c0, c1;
  long long ip;
  int z0, z1;
  bool valid;
};

// Thread -> (column, z range). DIM 3: block = 32 x 8 columns, blockIdx.z
// picks the z chunk. DIM 2: x from 32 lanes, (blockIdx.y, threadIdx.y) pick
// the chunk of rows (the slab axis is axis 1). DIM 1: one node per thread.
template <int DIM>
__device__ __forceinline__ Col<DIM> col_here(const Geom& g, int zc) {
  Col<DIM> c;
  if (DIM == 3) {
    c.c0 = blockIdx.x * FBX + threadIdx.x;
    c.c1 = blockIdx.y * FBY + threadIdx.y;
    c.z0 = blockIdx.z * zc;
    c.valid = c.c0 < g.n0 && c.c1 < g.n1;
    c.ip = (long long)c.c0 + (long long)g.n0 * c.c1;
  } else if (DIM == 2) {
    c.c0 = blockIdx.x * FBX + threadIdx.x;
    c.c1 = 0;
    c.z0 = (blockIdx.y * FBY + threadIdx.y) * zc;
    c.valid = c.c0 < g.n0;
    c.ip = c.c0;
  } else {
    c.c0 = c.c1 = 0;
    c.z0 = (blockIdx.x * FBY + threadIdx.y) * FBX + threadIdx.x;
    c.valid = true;
    c.ip = 0;
    zc = 1;
  }
  c.z1 = min(g.nzl, c.z0 + zc);
  c.valid = c.valid && c.z0 < c.z1;
  return c;
}

// Field value at local plane zz in [-1, nzl] of a column: interior, mirror
// at the global boundary (P/src/monodomain.cpp:85-86), or ghost plane.
__device__ __forceinline__ double zval(const double* __restrict__ f, const Geom& g,
                                       long long ip, int zz, const double* glo,
                                       const double* ghi) {
  if (zz >= 0 && zz < g.nzl) return __ldg(f + ip + g.plane * zz);
  int gz = zz + g.zoff;
  gz = gz < 0 ? 1 : (gz >= g.nzg ? g.nzg - 2 : gz);
  const int lz = gz - g.zoff;
  if (lz >= 0 && lz < g.nzl) return __ldg(f + ip + g.plane * lz);
  return lz < 0 ? __ldg(glo + ip) : __ldg(ghi + ip);
}

// In-plane neighbour offsets of a column (mirror at the boundaries).
template <int DIM>
struct Nbr {
  long long xm, xp, ym, yp;
};

template <int DIM>
__device__ __forceinline__ Nbr<DIM> nbr_of(const Geom& g, const Col<DIM>& c) {
  Nbr<DIM> o{0, 0, 0, 0};
  if (DIM >= 2) {
    o.xm = c.c0 > 0 ? -1 : 1;
    o.xp = c.c0 < g.n0 - 1 ? 1 : -1;
  }
  if (DIM == 3) {
    o.ym = c.c1 > 0 ? -(long long)g.n0 : (long long)g.n0;
    o.yp = c.c1 < g.n1 - 1 ? (long long)g.n0 : -(long long)g.n0;
  }
  return o;
}

// Scaled Laplacian with the column's z values in registers (FMA form;
// wc = -2 sum_a w_a).
template <int DIM>
__device__ __forceinline__ double lap_fast(const Geom& g, const double* __restrict__ f,
                                           long long i, const Nbr<DIM>& o, double vm,
                                           double vc, double vp) {
  double d = fma(g.wc, vc, g.w[DIM - 1] * (vp + vm));
  if (DIM >= 2) d = fma(g.w[0], __ldg(f + i + o.xm) + __ldg(f + i + o.xp), d);
  if (DIM == 3) d = fma(g.w[1], __ldg(f + i + o.ym) + __ldg(f + i + o.yp), d);
  return d;
}

template <int DIM>
__device__ __forceinline__ bool stim_col(const Geom& g, const Col<DIM>& c) {
  if (DIM == 3)
    return c.c0 >= g.st_lo[0] && c.c0 <= g.st_hi[0] && c.c1 >= g.st_lo[1] &&
           c.c1 <= g.st_hi[1];
  if (DIM == 2) return c.c0 >= g.st_lo[0] && c.c0 <= g.st_hi[0];
  return true;
}

template <int DIM>
__device__ __forceinline__ bool stim_col_xy(const Geom& g, int x, int y) {
  if (DIM == 3)
    return x >= g.st_lo[0] && x <= g.st_hi[0] && y >= g.st_lo[1] && y <= g.st_hi[1];
  return x >= g.st_lo[0] && x <= g.st_hi[0];
}

template <int DIM>
__device__ __forceinline__ bool stim_z(const Geom& g, int z) {
  const int zg = z + g.zoff;
  return zg >= g.st_lo[DIM - 1] && zg <= g.st_hi[DIM - 1];
}

// I_ion of HH (P/src/ionic.cpp:111-116), FMA form.
__device__ __forceinline__ double current_fast(double V, double m, double h, double n) {
  const double m2 = m * m;
  const double n2 = n * n;
  const double gna = kFC.gna * (m2 * m) * h;
  const double gk = kFC.gk * (n2 * n2);
  return fma(gna, V - kVNa, fma(gk, V - kVK, kFC.gl * (V - kFC.vl)));
}

// ---- cross-process halo protocol (Halo::sig_* / wait_*) -------------------
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Thread 0 spins until the ghost planes this block reads have arrived; the
// caller's __syncthreads() publishes that to the block. The spin is bounded
// (~10 s): a neighbour that never arrives (a rank died, or a caller drove
// linked slabs one at a time) records abort code 0 = protocol timeout
// instead of hanging the GPU.
__device__ __forceinline__ void halo_wait(const Halo& h, bool need_lo, bool need_hi) {
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    const long long t0 = clock64();
    const long long limit = 20000000000LL;  // cycles (~10 s at 2 GHz)
    bool late = false;
    if (need_lo && h.wait_lo)
      while (ld_acquire_sys(h.wait_lo) < h.expect_lo) {
        __nanosleep(200);
        if (clock64() - t0 > limit) { late = true; break; }
      }
    if (!late && need_hi && h.wait_hi)
      while (ld_acquire_sys(h.wait_hi) < h.expect_hi) {
        __nanosleep(200);
        if (clock64() - t0 > limit) { late = true; break; }
      }
    if (late && h.timeout_flag) atomicMin(h.timeout_flag, 0ull);
  }
}
// After all threads of the block wrote their boundary values.
__device__ __forceinline__ void halo_signal(const Halo& h, bool put_lo, bool put_hi) {
  if ((put_lo && h.sig_lo) || (put_hi && h.sig_hi)) {
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      __threadfence_system();
      if (put_lo && h.sig_lo) atomicAdd_system(h.sig_lo, 1ull);
      if (put_hi && h.sig_hi) atomicAdd_system(h.sig_hi, 1ull);
    }
  }
}

// Weighted form (wide d_1 halo): wlo / whi arrivals, one per plane stored.
__device__ __forceinline__ void halo_signal_w(const Halo& h, int wlo, int whi) {
  if ((wlo > 0 && h.sig_lo) || (whi > 0 && h.sig_hi)) {
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      __threadfence_system();
      if (wlo > 0 && h.sig_lo) atomicAdd_system(h.sig_lo, (unsigned long long)wlo);
      if (whi > 0 && h.sig_hi) atomicAdd_system(h.sig_hi, (unsigned long long)whi);
    }
  }
}

// Boundary planes a z-chunk [zb, ze) of a node kernel stores into the
// neighbours: planes z < zl go to plo + z * plane, planes z >= zh to
// phi + (z - zh) * plane. One plane (put_lo / put_hi) or, with h.kput, the
// K planes of the wide d_1 halo.
struct PutPlan {
  double* plo;
  double* phi;
  int zl, zh;
};
__device__ __forceinline__ PutPlan put_plan(const Halo& h, int nzl) {
  PutPlan pp;
  const int w = h.kput > 0 ? h.kput : 1;
  pp.plo = h.kput > 0 ? h.kput_lo : h.put_lo;
  pp.phi = h.kput > 0 ? h.kput_hi : h.put_hi;
  pp.zl = pp.plo ? w : 0;
  pp.zh = pp.phi ? nzl - w : 0x7fffffff;
  return pp;
}
// Arrivals of the chunk [zb, ze) per side (planes it stores).
__device__ __forceinline__ void put_signal(const Halo& h, const PutPlan& pp, int zb, int ze) {
  halo_signal_w(h, max(0, min(ze, pp.zl) - zb), max(0, ze - max(zb, pp.zh)));
}

__device__ __forceinline__ bool prologue(const unsigned long long* ev,
                                         unsigned long long floor, double* tab) {
  __shared__ int skip;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  if (tid == 0) skip = (*(volatile const unsigned long long*)ev) < floor;
  if (tab) load_exp_table(tab, tid, blockDim.x * blockDim.y);
  __syncthreads();
  return skip != 0;
}

__device__ __forceinline__ void block_gate_range(unsigned long long* slot,
                                                 unsigned long long lo,
                                                 unsigned long long hi) {
  __shared__ unsigned long long slo[kFThreads / 32], shi[kFThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  if ((tid & 31) == 0) {
    slo[tid >> 5] = lo;
    shi[tid >> 5] = hi;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kFThreads / 32; ++w) {
      lo = min(lo, slo[w]);
      hi = max(hi, shi[w]);
    }
    if (lo != ~0ull) atomicMin(slot, lo);
    if (hi != 0ull) atomicMax(slot + 1, hi);
  }
}

// Block min/max of the gate outputs (P/src/simulate.cpp:76-85): per-thread
// running min/max in double, one ordered-u64 atomic per block.
__device__ __forceinline__ void block_gate_range_d(unsigned long long* slot, double lo,
                                                   double hi, bool any) {
  block_gate_range(slot, any ? ord_of(lo) : ~0ull, any ? ord_of(hi) : 0ull);
}

// Per-node body shared by the z loop: computes the outputs of one node.
struct NodeOut {
  double o0, o1, o2, o3;
  double fs;
};

template <int DIM, int FIRST, int ION>
__device__ __forceinline__ NodeOut node_update(const Geom& g, const FastArgs& a,
                                               const double* __restrict__ tab, double vm,
                                               double vc, double vp, double xs, double ys,
                                               double z0, double z1, double z2, double stim,
                                               const double* __restrict__ q2) {
  double D = fma(g.wc, vc, g.w[DIM - 1] * (vp + vm));
  if (DIM >= 2) D = fma(g.w[0], xs, D);
  if (DIM == 3) D = fma(g.w[1], ys, D);
  double d0, d1, d2;
  if (fabs(vc - a.vmid) <= a.vfast) {
    hh_expeuler_fast(vc, z0, z1, z2, a.eta, tab, d0, d1, d2);
  } else {
    const Dgate dd = hh_expeuler_ref(vc, z0, z1, z2, a.eta);
    d0 = dd.d0;
    d1 = dd.d1;
    d2 = dd.d2;
  }
  const double fs = fma(-current_fast(vc, z0 + d0, z1 + d1, z2 + d2), g.inv_Cm, stim);
  const double fsum = D + fs;  // (f_F + f_S)(y_E) on V: inner stage 1
  double b0 = vc, b1 = z0, b2 = z1, b3 = z2;
  if (!FIRST) {
    b0 = fma(a.nu, vc, a.kappa * __ldg(q2));
    b1 = fma(a.nu, z0, a.kappa * __ldg(q2 + g.nn));
    b2 = fma(a.nu, z1, a.kappa * __ldg(q2 + 2 * g.nn));
    b3 = fma(a.nu, z2, a.kappa * __ldg(q2 + 3 * g.nn));
  }
  NodeOut r;
  r.o1 = fma(a.cG, d0, b1);
  r.o2 = fma(a.cG, d1, b2);
  r.o3 = fma(a.cG, d2, b3);
  r.o0 = ION ? a.mue1 * fsum : fma(a.cV, fsum, b0);
  r.fs = fs;
  return r;
}

template <int DIM, int FIRST, int ION, int SLOW = 1>
__device__ __forceinline__ NodeOut node_update_s(const Geom& g, const FastArgs& a,
                                                 const double* __restrict__ tab, double vm,
                                                 double vc, double vp, double xs, double ys,
                                                 double z0, double z1, double z2, double stim,
                                                 const double* q2s, int qstride) {
  double D = fma(g.wc, vc, g.w[DIM - 1] * (vp + vm));
  if (DIM >= 2) D = fma(g.w[0], xs, D);
  if (DIM == 3) D = fma(g.w[1], ys, D);
  double d0, d1, d2;
  if (!SLOW || fabs(vc - a.vmid) <= a.vfast) {
    hh_expeuler_fast(vc, z0, z1, z2, a.eta, tab, d0, d1, d2);
  } else {
    const Dgate dd = hh_expeuler_ref(vc, z0, z1, z2, a.eta);
    d0 = dd.d0;
    d1 = dd.d1;
    d2 = dd.d2;
  }
  const double fs = fma(-current_fast(vc, z0 + d0, z1 + d1, z2 + d2), g.inv_Cm, stim);
  const double fsum = D + fs;
  double b0 = vc, b1 = z0, b2 = z1, b3 = z2;
  if (!FIRST) {
    b0 = fma(a.nu, vc, a.kappa * q2s[0]);
    b1 = fma(a.nu, z0, a.kappa * q2s[qstride]);
    b2 = fma(a.nu, z1, a.kappa * q2s[2 * qstride]);
    b3 = fma(a.nu, z2, a.kappa * q2s[3 * qstride]);
  }
  NodeOut r;
  r.o1 = fma(a.cG, d0, b1);
  r.o2 = fma(a.cG, d1, b2);
  r.o3 = fma(a.cG, d2, b3);
  r.o0 = ION ? a.mue1 * fsum : fma(a.cV, fsum, b0);
  r.fs = fs;
  return r;
}

// Exact abort ordinal of a column whose outputs went non-finite: the
// reference checks inner stage 1 (y_E, f_F + f_S) before the outer stage
// (P/src/cheb.cpp:73-80, multirate.cpp:100-104). Rare path.
template <int DIM>
__device__ __noinline__ bool inner_nonfinite(const Geom& g, const Halo& h, const double* G,
                                             const Col<DIM>& c, const Nbr<DIM>& o, double eta) {
  bool inner = false;
  for (int z = c.z0; z < c.z1; ++z) {
    const long long j = c.ip + g.plane * z;
    const double V = zval(G, g, c.ip, z, h.lo, h.hi);
    double D = fma(g.wc, V, g.w[DIM - 1] * (zval(G, g, c.ip, z - 1, h.lo, h.hi) +
                                            zval(G, g, c.ip, z + 1, h.lo, h.hi)));
    if (DIM >= 2) D = fma(g.w[0], __ldg(G + j + o.xm) + __ldg(G + j + o.xp), D);
    if (DIM == 3) D = fma(g.w[1], __ldg(G + j + o.ym) + __ldg(G + j + o.yp), D);
    const double z0 = __ldg(G + g.nn + j), z1 = __ldg(G + 2 * g.nn + j),
                 z2 = __ldg(G + 3 * g.nn + j);
    const Dgate d = hh_expeuler_ref(V, z0, z1, z2, eta);
    const double y0 = z0 + d.d0, y1 = z1 + d.d1, y2 = z2 + d.d2;
    const double fs = -current_fast(V, y0, y1, y2) * g.inv_Cm;
    inner |= !(finite_hi(D + fs) && finite_hi(y0) && finite_hi(y1) && finite_hi(y2));
    for (int q = 0; q < g.naux; ++q) {  // aux rows of u_1: z + mu'_1 eta g_S(V, z)
      const double za = __ldg(G + (4 + q) * g.nn + j);
      inner |= !(finite_hi(za) && finite_hi(aux_rate_fast(q, V, za)));
    }
  }
  return inner;
}

// ---------------------------------------------------------------------------
// k_node_fast: m == 1 (ION = 0, one HBM pass per outer stage) and the first
// inner stage of m >= 2 (ION = 1: gate rows of g_j, fs, u_1).
// ---------------------------------------------------------------------------
#ifndef EMRKC_NODE_MINBLOCKS
#define EMRKC_NODE_MINBLOCKS 1
#endif
#ifndef EMRKC_NODE_UNROLL
#define EMRKC_NODE_UNROLL 2
#endif
constexpr int kNodeUnroll = EMRKC_NODE_UNROLL;
template <int DIM, int FIRST, int ION>
__global__ void __launch_bounds__(kFThreads, EMRKC_NODE_MINBLOCKS)
    k_node_fast(const Geom g, const Halo h, const FastArgs a) {
  __shared__ double tab[256];
  const int bz0 = (DIM == 3 ? blockIdx.z * a.zc : blockIdx.y * FBY * a.zc);
  const int bz1 = (DIM == 3 ? bz0 + a.zc : bz0 + FBY * a.zc);
  halo_wait(h, bz0 == 0, bz1 >= g.nzl);
  if (prologue(a.event, level_floor(a.code_base, a.j, a.m, 1), tab)) {  // aborted earlier: still release the neighbours
    halo_signal(h, bz0 == 0, bz1 >= g.nzl);
    return;
  }
  const Col<DIM> c = col_here<DIM>(g, a.zc);
  bool bad = false, guard = false, any = false;
  double glo = 2.0, ghi = -1.0;
  if (c.valid) {
    const Nbr<DIM> o = nbr_of<DIM>(g, c);
    const bool scol = stim_col<DIM>(g, c);
    const long long plane = g.plane, nn = g.nn;
    const double* __restrict__ G = a.g1;
    const long long i0 = c.ip + plane * c.z0;
    const double* pv = G + i0;           // V of g_{j-1} at (column, z)
    const double* pz = G + nn + i0;      // gate 0 (gates 1, 2 at +nn, +2nn)
    double* po = a.out + i0;             // g_j
    const double* q2 = FIRST ? nullptr : a.g2 + i0;
    double* pu = ION ? a.u1 + i0 : nullptr;
    double vm = zval(G, g, c.ip, c.z0 - 1, h.lo, h.hi);
    double vc = __ldg(pv);
#pragma unroll kNodeUnroll
    for (int z = c.z0; z < c.z1; ++z) {
      const double vp = (z + 1 < g.nzl) ? __ldg(pv + plane)
                                        : zval(G, g, c.ip, z + 1, h.lo, h.hi);
      double xs = 0.0, ys = 0.0;
      if (DIM >= 2) xs = __ldg(pv + o.xm) + __ldg(pv + o.xp);
      if (DIM == 3) ys = __ldg(pv + o.ym) + __ldg(pv + o.yp);
      const double z0 = __ldg(pz), z1 = __ldg(pz + nn), z2 = __ldg(pz + 2 * nn);
      const double stim = (scol && stim_z<DIM>(g, z)) ? a.stim : 0.0;
      const NodeOut r = node_update<DIM, FIRST, ION>(g, a, tab, vm, vc, vp, xs, ys, z0, z1,
                                                     z2, stim, q2);
      po[nn] = r.o1;
      po[2 * nn] = r.o2;
      po[3 * nn] = r.o3;
      if (ION) {
        *pu = r.o0;  // d_1
        pu += plane;
      } else {
        *po = r.o0;
        guard |= !(fabs(r.o0) <= 1e6);  // also a non-finite V
      }
      bad |= !(finite_hi(r.o0) && finite_hi(r.o1) && finite_hi(r.o2) && finite_hi(r.o3));
      if (z == 0 && h.put_lo) h.put_lo[c.ip] = r.o0;
      if (z == g.nzl - 1 && h.put_hi) h.put_hi[c.ip] = r.o0;
      if (a.last) {
        glo = fmin(glo, fmin(r.o1, fmin(r.o2, r.o3)));
        ghi = fmax(ghi, fmax(r.o1, fmax(r.o2, r.o3)));
        any = true;
      }
      vm = vc;
      vc = vp;
      pv += plane;
      pz += plane;
      po += plane;
      if (!FIRST) q2 += plane;
    }
    if (bad && !a.exex) {  // EXEX-RL never throws NumericalAbort
      const bool inner = inner_nonfinite<DIM>(g, h, G, c, o, a.eta);
      atomicMin(a.event, a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1)) +
                             (inner ? 1 : a.m + 1));
    }
  }
  if (!ION && a.last && guard)
    atomicMin(a.event, a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
  if (a.last) block_gate_range_d(a.gate_slot, glo, ghi, any);
  halo_signal(h, bz0 == 0, bz1 >= g.nzl);
}

// ---------------------------------------------------------------------------
// k_node_pipe: the node kernel with its planes staged through shared memory
// by cp.async (LDGSTS), two planes ahead of the compute. A block owns a
// TX x TY column tile and walks zc planes; each plane stage holds the V tile
// with a one-cell halo (mirror cells resolved at load time, so the compute
// has no boundary logic) and the tile's gate values. Ring depths: V 5
// (planes p-1, p, p+1 read while p+2 lands), gates 4 — each stage is
// rewritten only after a __syncthreads separates it from its last reader.
// ---------------------------------------------------------------------------
template <int DIM>
struct PipeTile {
  static constexpr int TX = DIM == 3 ? 32 : 128;
  static constexpr int TY = DIM == 3 ? 4 : 1;
  static constexpr int HX = TX + 2;
  static constexpr int HY = DIM == 3 ? TY + 2 : 1;
  static constexpr int VT = HX * HY;  // V cells per stage
  static constexpr int NT = TX * TY;  // threads = tile columns
};
constexpr int kRV = 8;  // power of two >= 5
constexpr int kRG = 4;

template <int DIM, int FIRST>
constexpr size_t pipe_smem_bytes() {  // dynamic part (k_node_persist adds the table)
  using T = PipeTile<DIM>;
  return sizeof(double) * (256 + kRV * T::VT + kRG * 3 * T::NT + (FIRST ? 0 : kRG * 4 * T::NT));
}

__device__ __forceinline__ void cp_async8(unsigned sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Source of V for local plane zz in [-1, nzl]: state plane, mirror plane at
// the global boundary (P/src/monodomain.cpp:85-86), or ghost plane.
__device__ __forceinline__ const double* vplane(const Geom& g, const Halo& h,
                                                const double* G, int zz) {
  if (zz >= 0 && zz < g.nzl) return G + g.plane * zz;
  int gz = zz + g.zoff;
  gz = gz < 0 ? 1 : (gz >= g.nzg ? g.nzg - 2 : gz);
  const int lz = gz - g.zoff;
  if (lz >= 0 && lz < g.nzl) return G + g.plane * lz;
  return lz < 0 ? h.lo : h.hi;
}

// In-plane offset of halo cell c of a tile (mirror at the grid edge; cells
// past the far edge clamp to a valid node, their values are never read).
template <int DIM>
__device__ __forceinline__ long long halo_offset(const Geom& g, int x0, int y0, int c) {
  using T = PipeTile<DIM>;
  const int hx = c % T::HX, hy = c / T::HX;
  int gx = x0 + hx - 1;
  gx = gx < 0 ? 1 : (gx >= g.n0 ? max(g.n0 - 2, 0) : gx);
  int gy = 0;
  if (DIM == 3) {
    gy = y0 + hy - 1;
    gy = gy < 0 ? 1 : (gy >= g.n1 ? max(g.n1 - 2, 0) : gy);
  }
  return gx + (long long)g.n0 * gy;
}

#ifndef EMRKC_PIPE_MINBLOCKS
#define EMRKC_PIPE_MINBLOCKS 5
#endif

template <int DIM, int FIRST, int ION>
__global__ void __launch_bounds__(PipeTile<DIM>::NT, EMRKC_PIPE_MINBLOCKS)
    k_node_pipe(const Geom g, const Halo h, const FastArgs a) {
  using T = PipeTile<DIM>;
  extern __shared__ double smem[];
  __shared__ double tab[256];                     // static: immediate LDS offsets
  double* vst = smem;                             // [kRV][VT]
  double* gst = vst + kRV * T::VT;                // [kRG][3][NT]
  double* g2s = gst + kRG * 3 * T::NT;            // [kRG][4][NT] (!FIRST)
  const int t = threadIdx.x;
  pdl_launch_dependents();
  pdl_wait();
  {
    const int zb0 = (DIM == 3 ? blockIdx.z : blockIdx.y) * a.zc;
    halo_wait(h, zb0 == 0, zb0 + a.zc >= g.nzl);
    if (h.wait_lo || h.wait_hi) __syncthreads();
  }
  __shared__ int skip;
  if (t == 0) skip = (*(volatile const unsigned long long*)a.event) < level_floor(a.code_base, a.j, a.m, 1);
  {
    // exp table rides in the first cp.async group with the first planes
    const unsigned st = (unsigned)__cvta_generic_to_shared(tab);
    for (int j = t; j < 256; j += T::NT) cp_async8(st + 8u * j, kExp2Tab256 + j);
  }
  const int tx = t % T::TX, ty = t / T::TX;
  const int x0 = blockIdx.x * T::TX;
  const int y0 = DIM == 3 ? blockIdx.y * T::TY : 0;
  const int zb = (DIM == 3 ? blockIdx.z : blockIdx.y) * a.zc;
  const int ze = min(g.nzl, zb + a.zc);
  const int cx = x0 + tx, cy = y0 + ty;
  const bool valid = cx < g.n0 && (DIM == 2 || cy < g.n1);
  const long long ip = valid ? (long long)cx + (long long)g.n0 * cy : 0;
  const long long nn = g.nn, plane = g.plane;
  const double* G = a.g1;
  // per-thread copy plan, resolved once: halo cells t and t + NT of every V
  // stage, the thread's own column for the gates (and g_{j-2})
  const long long voff0 = halo_offset<DIM>(g, x0, y0, t);
  const bool has1 = t + T::NT < T::VT;
  const long long voff1 = has1 ? halo_offset<DIM>(g, x0, y0, t + T::NT) : 0;
  const double* vsrc0 = G + voff0;  // + plane * zz for an interior plane
  const double* vsrc1 = G + voff1;
  const unsigned sv0 = (unsigned)__cvta_generic_to_shared(vst) + 8u * t;
  const unsigned sg0 = (unsigned)__cvta_generic_to_shared(gst) + 8u * t;
  const unsigned sq0 = (unsigned)__cvta_generic_to_shared(g2s) + 8u * t;
  const double* gz0 = G + nn + ip;    // gate columns
  const double* qz0 = FIRST ? nullptr : a.g2 + ip;

  auto load_plane = [&](int zz) {
    const unsigned sv = sv0 + 8u * T::VT * ((zz - zb + 1) & (kRV - 1));
    if (zz >= 0 && zz < g.nzl) {
      const long long o = plane * zz;
      cp_async8(sv, vsrc0 + o);
      if (has1) cp_async8(sv + 8u * T::NT, vsrc1 + o);
    } else {  // outside the slab: mirror plane or ghost plane (first/last chunk only)
      const double* vp = vplane(g, h, G, zz);
      cp_async8(sv, vp + voff0);
      if (has1) cp_async8(sv + 8u * T::NT, vp + voff1);
    }
    if (zz >= zb && zz < ze) {
      const unsigned s = (unsigned)((zz - zb) & (kRG - 1));
      const unsigned sg = sg0 + 8u * 3 * T::NT * s;
      const double* gp = gz0 + plane * zz;
      cp_async8(sg, gp);
      cp_async8(sg + 8u * T::NT, gp + nn);
      cp_async8(sg + 16u * T::NT, gp + 2 * nn);
      if (!FIRST) {
        const unsigned sq = sq0 + 8u * 4 * T::NT * s;
        const double* qp = qz0 + plane * zz;
        cp_async8(sq, qp);
        cp_async8(sq + 8u * T::NT, qp + nn);
        cp_async8(sq + 16u * T::NT, qp + 2 * nn);
        cp_async8(sq + 24u * T::NT, qp + 3 * nn);
      }
    }
    cp_commit();
  };

  load_plane(zb - 1);
  load_plane(zb);
  load_plane(zb + 1);
  __syncthreads();  // publishes `skip`
  const bool skipped = skip != 0;
  // stimulus rows of this column: z in [zs0, zs1] (P/src/monodomain.cpp:151-158)
  int zs0 = 1, zs1 = 0;
  if (valid && stim_col_xy<DIM>(g, cx, cy)) {
    zs0 = g.st_lo[DIM - 1] - g.zoff;
    zs1 = g.st_hi[DIM - 1] - g.zoff;
  }
  bool bad = false, guard = false;
  unsigned slow_mask = 0;  // planes (z - zb < 32) left to the reference path
  double glo = 2.0, ghi = -1.0;
  const int cell = (DIM == 3 ? (ty + 1) * T::HX : 0) + tx + 1;
  double* po = a.out + ip + plane * zb;
  double* pu = ION ? a.u1 + ip + plane * zb : nullptr;
  for (int z = zb; z < ze && !skipped; ++z) {
    if (z + 2 <= ze) {
      load_plane(z + 2);
    } else {
      cp_commit();  // keep the group count uniform
    }
    cp_wait<1>();
    __syncthreads();
    const int p = z - zb + 1;
    const double* V0 = vst + (p & (kRV - 1)) * T::VT;
    const double vc = V0[cell];
    const double vm = vst[((p - 1) & (kRV - 1)) * T::VT + cell];
    const double vp = vst[((p + 1) & (kRV - 1)) * T::VT + cell];
    double xs = 0.0, ys = 0.0;
    if (DIM >= 2) xs = V0[cell - 1] + V0[cell + 1];
    if (DIM == 3) ys = V0[cell - T::HX] + V0[cell + T::HX];
    const double* G0 = gst + ((z - zb) & (kRG - 1)) * 3 * T::NT + t;
    const double z0 = G0[0], z1 = G0[T::NT], z2 = G0[2 * T::NT];
    // |V| beyond the fast path's range (or non-finite): deferred to the
    // reference-order path after the loop, so the hot loop has no call
    const bool fast = fabs(vc - a.vmid) <= a.vfast;
    if (!fast) slow_mask |= 1u << (z - zb);
    NodeOut r = node_update_s<DIM, FIRST, ION, 0>(
        g, a, tab, vm, vc, vp, xs, ys, z0, z1, z2, 0.0,
        g2s + ((z - zb) & (kRG - 1)) * 4 * T::NT + t, T::NT);
    if (z >= zs0 && z <= zs1) {  // stimulus (rare): fs gains +stim
      if (ION) r.o0 = fma(a.mue1, a.stim, r.o0);
      else r.o0 = fma(a.cV, a.stim, r.o0);
    }
    if (valid && fast) {
      po[nn] = r.o1;
      po[2 * nn] = r.o2;
      po[3 * nn] = r.o3;
      if (ION) {
        *pu = r.o0;  // d_1
      } else {
        *po = r.o0;
        guard |= !(fabs(r.o0) <= 1e6);  // also a non-finite V
      }
      // one finiteness test per node: a non-finite output poisons the sum
      bad |= !finite_hi((r.o0 + r.o1) + (r.o2 + r.o3));
      if (z == 0 && h.put_lo) h.put_lo[ip] = r.o0;
      if (z == g.nzl - 1 && h.put_hi) h.put_hi[ip] = r.o0;
      if (a.last) {  // std::min / std::max per value (NaN skipped), select form
        glo = r.o1 < glo ? r.o1 : glo;
        ghi = ghi < r.o1 ? r.o1 : ghi;
        glo = r.o2 < glo ? r.o2 : glo;
        ghi = ghi < r.o2 ? r.o2 : ghi;
        glo = r.o3 < glo ? r.o3 : glo;
        ghi = ghi < r.o3 ? r.o3 : ghi;
      }
    }
    po += plane;
    if (ION) pu += plane;
  }
  cp_wait<0>();
  if (!skipped && valid && slow_mask) {
    // deferred nodes: reference-order ionic path, inputs from global memory
    const Nbr<DIM> o = nbr_of<DIM>(g, Col<DIM>{cx, cy, ip, zb, ze, true});
    for (int z = zb; z < ze; ++z) {
      if (!(slow_mask >> (z - zb) & 1u)) continue;
      const long long i = ip + plane * z;
      const double vc = __ldg(G + i);
      const double vm = zval(G, g, ip, z - 1, h.lo, h.hi);
      const double vp = zval(G, g, ip, z + 1, h.lo, h.hi);
      double xs = 0.0, ys = 0.0;
      if (DIM >= 2) xs = __ldg(G + i + o.xm) + __ldg(G + i + o.xp);
      if (DIM == 3) ys = __ldg(G + i + o.ym) + __ldg(G + i + o.yp);
      const double stim = (z >= zs0 && z <= zs1) ? a.stim : 0.0;
      double q[4] = {0.0, 0.0, 0.0, 0.0};
      if (!FIRST)
        for (int f = 0; f < 4; ++f) q[f] = __ldg(a.g2 + f * nn + i);
      const NodeOut r = node_update_s<DIM, FIRST, ION, 1>(
          g, a, tab, vm, vc, vp, xs, ys, __ldg(G + nn + i), __ldg(G + 2 * nn + i),
          __ldg(G + 3 * nn + i), stim, q, 1);
      a.out[nn + i] = r.o1;
      a.out[2 * nn + i] = r.o2;
      a.out[3 * nn + i] = r.o3;
      if (ION) {
        a.u1[i] = r.o0;
      } else {
        a.out[i] = r.o0;
        guard |= !(fabs(r.o0) <= 1e6);  // also a non-finite V
      }
      bad |= !finite_hi((r.o0 + r.o1) + (r.o2 + r.o3));
      if (z == 0 && h.put_lo) h.put_lo[ip] = r.o0;
      if (z == g.nzl - 1 && h.put_hi) h.put_hi[ip] = r.o0;
      if (a.last) {
        glo = fmin(glo, fmin(r.o1, fmin(r.o2, r.o3)));
        ghi = fmax(ghi, fmax(r.o1, fmax(r.o2, r.o3)));
      }
    }
  }
  halo_signal(h, zb == 0, ze >= g.nzl);  // also when skipping: release the neighbours
  if (skipped) return;
  if (bad && !a.exex) {  // EXEX-RL never throws NumericalAbort
    Col<DIM> c;
    c.c0 = cx;
    c.c1 = cy;
    c.ip = ip;
    c.z0 = zb;
    c.z1 = ze;
    c.valid = true;
    const bool inner = inner_nonfinite<DIM>(g, h, G, c, nbr_of<DIM>(g, c), a.eta);
    atomicMin(a.event, a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1)) +
                           (inner ? 1 : a.m + 1));
  }
  if (!ION && a.last && guard)
    atomicMin(a.event, a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
  if (a.last) block_gate_range_d(a.gate_slot, glo, ghi, valid && ze > zb);
}

#if EMRKC_EXPERIMENTAL  // k_node_persist: measured slower than k_node_tma
// Loader state of one work item (prepared outside the inner loop).
struct PLoad {
  long long voff0, voff1;   // halo cells t and t + NT of the tile
  const double* gcol;       // gate 0 of the thread's column
  const double* qcol;       // g_{j-2} of the thread's column
  int zz, zb, ze;           // next plane to load, item planes
  int live;                 // 0: past the last item
};

template <int DIM>
__device__ __forceinline__ void item_geom(int it, int nchunk, int tiles_x, int zc, int nzl,
                                          int& x0, int& y0, int& zb, int& ze) {
  using T = PipeTile<DIM>;
  const int chunk = it % nchunk;
  const int tile = it / nchunk;
  x0 = (tile % tiles_x) * T::TX;
  y0 = DIM == 3 ? (tile / tiles_x) * T::TY : 0;
  zb = chunk * zc;
  ze = min(nzl, zb + zc);
}

template <int DIM, int FIRST>
__device__ __noinline__ PLoad prep_item(const Geom& g, const Halo& h, const FastArgs& a, int it,
                                        int items, int nchunk, int tiles_x, int t) {
  using T = PipeTile<DIM>;
  PLoad L;
  L.live = it < items;
  if (!L.live) {
    L.voff0 = L.voff1 = 0;
    L.gcol = L.qcol = nullptr;
    L.zz = L.zb = L.ze = 0;
    return L;
  }
  int x0, y0;
  item_geom<DIM>(it, nchunk, tiles_x, a.zc, g.nzl, x0, y0, L.zb, L.ze);
  L.zz = L.zb - 1;
  L.voff0 = halo_offset<DIM>(g, x0, y0, t);
  L.voff1 = (t + T::NT < T::VT) ? halo_offset<DIM>(g, x0, y0, t + T::NT) : 0;
  const int tx = t % T::TX, ty = t / T::TX;
  const int cx = x0 + tx, cy = y0 + ty;
  const bool v = cx < g.n0 && (DIM == 2 || cy < g.n1);
  const long long ip = v ? (long long)cx + (long long)g.n0 * cy : 0;
  L.gcol = a.g1 + g.nn + ip;
  L.qcol = FIRST ? nullptr : a.g2 + ip;
  return L;
}

template <int DIM, int FIRST, int ION>
__global__ void __launch_bounds__(PipeTile<DIM>::NT, EMRKC_PIPE_MINBLOCKS)
    k_node_persist(const Geom g, const Halo h, const FastArgs a, const int items,
                   const int tiles_x) {
  using T = PipeTile<DIM>;
  extern __shared__ double smem[];
  double* tab = smem;
  double* vst = smem + 256;                       // [kRV][VT]
  double* gst = vst + kRV * T::VT;                // [kRG][3][NT]
  double* g2s = gst + kRG * 3 * T::NT;            // [kRG][4][NT] (!FIRST)
  const int t = threadIdx.x;
  __shared__ int skip;
  if (t == 0) skip = (*(volatile const unsigned long long*)a.event) < level_floor(a.code_base, a.j, a.m, 1);
  {
    const unsigned st = (unsigned)__cvta_generic_to_shared(tab);
    for (int j = t; j < 256; j += T::NT) cp_async8(st + 8u * j, kExp2Tab256 + j);
    cp_commit();
  }
  const int tx = t % T::TX, ty = t / T::TX;
  const int nchunk = (g.nzl + a.zc - 1) / a.zc;
  const long long nn = g.nn, plane = g.plane;
  const double* G = a.g1;
  const unsigned sv0 = (unsigned)__cvta_generic_to_shared(vst) + 8u * t;
  const unsigned sg0 = (unsigned)__cvta_generic_to_shared(gst) + 8u * t;
  const unsigned sq0 = (unsigned)__cvta_generic_to_shared(g2s) + 8u * t;
  const bool has1 = t + T::NT < T::VT;
  const int cell = (DIM == 3 ? (ty + 1) * T::HX : 0) + tx + 1;
  auto faces = [&](const PLoad& L, bool& lo, bool& hi) {
    lo = L.live && L.zb == 0 && h.wait_lo;
    hi = L.live && L.ze >= g.nzl && h.wait_hi;
  };

  int q = 0, c = 0;  // V / gate load sequence numbers
  // issues the next plane of L (one commit group per call); returns false
  // when L is exhausted (the caller switches L to the next item)
  auto issue = [&](PLoad& L) {
    const unsigned sv = sv0 + 8u * T::VT * (q & (kRV - 1));
    const double* vp = vplane(g, h, G, L.zz);
    cp_async8(sv, vp + L.voff0);
    if (has1) cp_async8(sv + 8u * T::NT, vp + L.voff1);
    if (L.zz >= L.zb && L.zz < L.ze) {
      const unsigned s = (unsigned)(c & (kRG - 1));
      const unsigned sg = sg0 + 8u * 3 * T::NT * s;
      const double* gp = L.gcol + plane * L.zz;
      cp_async8(sg, gp);
      cp_async8(sg + 8u * T::NT, gp + nn);
      cp_async8(sg + 16u * T::NT, gp + 2 * nn);
      if (!FIRST) {
        const unsigned sq = sq0 + 8u * 4 * T::NT * s;
        const double* qp = L.qcol + plane * L.zz;
        cp_async8(sq, qp);
        cp_async8(sq + 8u * T::NT, qp + nn);
        cp_async8(sq + 16u * T::NT, qp + 2 * nn);
        cp_async8(sq + 24u * T::NT, qp + 3 * nn);
      }
      ++c;
    }
    ++q;
    ++L.zz;
  };

  PLoad ld = prep_item<DIM, FIRST>(g, h, a, blockIdx.x, items, nchunk, tiles_x, t);
  {
    bool lo, hi;
    faces(ld, lo, hi);
    if (lo || hi) {
      halo_wait(h, lo, hi);
      __syncthreads();
    }
  }
  PLoad nx = prep_item<DIM, FIRST>(g, h, a, blockIdx.x + gridDim.x, items, nchunk, tiles_x, t);
  for (int r = 0; r < 3; ++r) {
    if (ld.live) issue(ld);
    cp_commit();
  }
  bool bad = false, guard = false, any = false;
  double glo = 2.0, ghi = -1.0;
  int cq = 1, cc = 0;  // sequence numbers of the plane being computed
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    int x0, y0, zb, ze;
    item_geom<DIM>(it, nchunk, tiles_x, a.zc, g.nzl, x0, y0, zb, ze);
    const int cx = x0 + tx, cy = y0 + ty;
    const bool valid = cx < g.n0 && (DIM == 2 || cy < g.n1);
    const long long ip = valid ? (long long)cx + (long long)g.n0 * cy : 0;
    const bool scol = valid && stim_col_xy<DIM>(g, cx, cy);
    double* po = a.out + ip + plane * zb;
    double* pu = ION ? a.u1 + ip + plane * zb : nullptr;
    unsigned slow_mask = 0;
    for (int z = zb; z < ze; ++z) {
      // keep the loader two planes ahead; it crosses into the next item
      // (prepared outside this loop) when the current one is exhausted
      if (ld.zz > ld.ze) {
        ld = nx;
        nx.live = 0;
      }
      if (ld.live) issue(ld);
      cp_commit();
      cp_wait<1>();
      __syncthreads();
      if (skip) break;
      const double* V0 = vst + (cq & (kRV - 1)) * T::VT;
      const double vc = V0[cell];
      const double vm = vst[((cq - 1) & (kRV - 1)) * T::VT + cell];
      const double vp = vst[((cq + 1) & (kRV - 1)) * T::VT + cell];
      double xs = 0.0, ys = 0.0;
      if (DIM >= 2) xs = V0[cell - 1] + V0[cell + 1];
      if (DIM == 3) ys = V0[cell - T::HX] + V0[cell + T::HX];
      const double* G0 = gst + (cc & (kRG - 1)) * 3 * T::NT + t;
      const double z0 = G0[0], z1 = G0[T::NT], z2 = G0[2 * T::NT];
      const double stim = (scol && stim_z<DIM>(g, z)) ? a.stim : 0.0;
      const bool fast = fabs(vc - a.vmid) <= a.vfast;
      if (!fast) slow_mask |= 1u << (z - zb);
      const NodeOut rr = node_update_s<DIM, FIRST, ION, 0>(
          g, a, tab, vm, vc, vp, xs, ys, z0, z1, z2, stim,
          g2s + (cc & (kRG - 1)) * 4 * T::NT + t, T::NT);
      if (valid && fast) {
        po[nn] = rr.o1;
        po[2 * nn] = rr.o2;
        po[3 * nn] = rr.o3;
        if (ION) {
          *pu = rr.o0;
        } else {
          *po = rr.o0;
          guard |= !(fabs(rr.o0) <= 1e6);  // also a non-finite V
        }
        bad |= !finite_hi((rr.o0 + rr.o1) + (rr.o2 + rr.o3));
        if (z == 0 && h.put_lo) h.put_lo[ip] = rr.o0;
        if (z == g.nzl - 1 && h.put_hi) h.put_hi[ip] = rr.o0;
        if (a.last) {  // std::min / std::max per value (NaN skipped), select form
          glo = rr.o1 < glo ? rr.o1 : glo;
          ghi = ghi < rr.o1 ? rr.o1 : ghi;
          glo = rr.o2 < glo ? rr.o2 : glo;
          ghi = ghi < rr.o2 ? rr.o2 : ghi;
          glo = rr.o3 < glo ? rr.o3 : glo;
          ghi = ghi < rr.o3 ? rr.o3 : ghi;
          any = true;
        }
      }
      po += plane;
      if (ION) pu += plane;
      ++cq;
      ++cc;
    }
    if (skip) {  // keep the neighbour protocol alive, then stop
      for (int j = it; j < items; j += gridDim.x) {
        int a0, a1, b0, b1;
        item_geom<DIM>(j, nchunk, tiles_x, a.zc, g.nzl, a0, a1, b0, b1);
        halo_signal(h, b0 == 0, b1 >= g.nzl);
      }
      break;
    }
    cq += 2;  // past this item's plane ze and the next item's zb - 1
    // the two extra planes of the next item (its zb - 1 and zb)
    for (int r = 0; r < 2; ++r) {
      if (ld.zz > ld.ze) {
        ld = nx;
        nx.live = 0;
      }
      if (ld.live) issue(ld);
      cp_commit();
    }
    if (valid && slow_mask) {
      // deferred nodes: reference-order ionic path from global memory
      const Nbr<DIM> o = nbr_of<DIM>(g, Col<DIM>{cx, cy, ip, zb, ze, true});
      for (int z = zb; z < ze; ++z) {
        if (!(slow_mask >> (z - zb) & 1u)) continue;
        const long long i = ip + plane * z;
        const double vc = __ldg(G + i);
        double xs = 0.0, ys = 0.0;
        if (DIM >= 2) xs = __ldg(G + i + o.xm) + __ldg(G + i + o.xp);
        if (DIM == 3) ys = __ldg(G + i + o.ym) + __ldg(G + i + o.yp);
        double qv[4] = {0.0, 0.0, 0.0, 0.0};
        if (!FIRST)
          for (int f = 0; f < 4; ++f) qv[f] = __ldg(a.g2 + f * nn + i);
        const NodeOut rr = node_update_s<DIM, FIRST, ION, 1>(
            g, a, tab, zval(G, g, ip, z - 1, h.lo, h.hi), vc, zval(G, g, ip, z + 1, h.lo, h.hi),
            xs, ys, __ldg(G + nn + i), __ldg(G + 2 * nn + i), __ldg(G + 3 * nn + i),
            (scol && stim_z<DIM>(g, z)) ? a.stim : 0.0, qv, 1);
        a.out[nn + i] = rr.o1;
        a.out[2 * nn + i] = rr.o2;
        a.out[3 * nn + i] = rr.o3;
        if (ION) {
          a.u1[i] = rr.o0;
        } else {
          a.out[i] = rr.o0;
          guard |= !(fabs(rr.o0) <= 1e6);  // also a non-finite V
        }
        bad |= !finite_hi((rr.o0 + rr.o1) + (rr.o2 + rr.o3));
        if (z == 0 && h.put_lo) h.put_lo[ip] = rr.o0;
        if (z == g.nzl - 1 && h.put_hi) h.put_hi[ip] = rr.o0;
        if (a.last) {
          glo = fmin(glo, fmin(rr.o1, fmin(rr.o2, rr.o3)));
          ghi = fmax(ghi, fmax(rr.o1, fmax(rr.o2, rr.o3)));
          any = true;
        }
      }
    }
    halo_signal(h, zb == 0, ze >= g.nzl);
    if (bad && !a.exex) {  // EXEX-RL never throws NumericalAbort
      const bool inner = valid && inner_nonfinite<DIM>(g, h, G, Col<DIM>{cx, cy, ip, zb, ze, true},
                                                       nbr_of<DIM>(g, Col<DIM>{cx, cy, ip, zb, ze, true}),
                                                       a.eta);
      atomicMin(a.event, a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1)) +
                             (inner ? 1 : a.m + 1));
      bad = false;
    }
    // prepare the item after the one the loader is on (outside the hot loop)
    if (!nx.live) {
      const int nxt = it + 2 * gridDim.x;
      nx = prep_item<DIM, FIRST>(g, h, a, nxt, items, nchunk, tiles_x, t);
      bool lo, hi;
      faces(nx, lo, hi);
      if (lo || hi) {
        halo_wait(h, lo, hi);
        __syncthreads();
      }
    }
  }
  cp_wait<0>();
  if (skip) return;
  if (!ION && a.last && guard)
    atomicMin(a.event, a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
  if (a.last) block_gate_range_d(a.gate_slot, glo, ghi, any);
}
#endif  // EMRKC_EXPERIMENTAL

// ---------------------------------------------------------------------------
// k_vin_pipe: the V-only inner stage with the same cp.async plane ring as
// k_node_pipe. Stencil field d_{k-1} with halo; pointwise d_{k-2}, d_1 and,
// on the last stage, V of g_{j-1} (and g_{j-2}).
// ---------------------------------------------------------------------------
template <int DIM>
constexpr size_t vin_smem_bytes() {
  using T = PipeTile<DIM>;
  return sizeof(double) * (kRV * T::VT + kRG * 4 * T::NT);
}

template <int DIM, int LAST, int FIRST>
__global__ void __launch_bounds__(PipeTile<DIM>::NT, 7)
    k_vin_pipe(const Geom g, const Halo h, const FastInnerArgs a) {
  using T = PipeTile<DIM>;
  extern __shared__ double smem[];
  double* vst = smem;                  // [kRV][VT]   d_{k-1} with halo
  double* cst = vst + kRV * T::VT;     // [kRG][4][NT] d1, d_{k-2}, V1, V2
  const int t = threadIdx.x;
  pdl_launch_dependents();
  pdl_wait();
  {
    const int zb0 = (DIM == 3 ? blockIdx.z : blockIdx.y) * a.zc;
    halo_wait(h, zb0 == 0, zb0 + a.zc >= g.nzl);
    if (h.wait_lo || h.wait_hi) __syncthreads();
  }
  __shared__ int skip;
  if (t == 0) skip = (*(volatile const unsigned long long*)a.event) < level_floor(a.code_base, a.j, a.m, a.k);
  const int tx = t % T::TX, ty = t / T::TX;
  const int x0 = blockIdx.x * T::TX;
  const int y0 = DIM == 3 ? blockIdx.y * T::TY : 0;
  const int zb = (DIM == 3 ? blockIdx.z : blockIdx.y) * a.zc;
  const int ze = min(g.nzl, zb + a.zc);
  const int cx = x0 + tx, cy = y0 + ty;
  const bool valid = cx < g.n0 && (DIM == 2 || cy < g.n1);
  const long long ip = valid ? (long long)cx + (long long)g.n0 * cy : 0;
  const long long plane = g.plane;
  const double* U = a.um1;
  const long long voff0 = halo_offset<DIM>(g, x0, y0, t);
  const bool has1 = t + T::NT < T::VT;
  const long long voff1 = has1 ? halo_offset<DIM>(g, x0, y0, t + T::NT) : 0;
  const unsigned sv0 = (unsigned)__cvta_generic_to_shared(vst) + 8u * t;
  const unsigned sc0 = (unsigned)__cvta_generic_to_shared(cst) + 8u * t;
  const bool has2 = a.um2 != nullptr;
  const bool d1_is_u = a.um1 == a.d1;  // k == 2: d_1 is the stencil field itself

  const double* usrc0 = U + voff0;
  const double* usrc1 = U + voff1;
  auto load_plane = [&](int zz) {
    const unsigned sv = sv0 + 8u * T::VT * ((zz - zb + 1) & (kRV - 1));
    if (zz >= 0 && zz < g.nzl) {
      const long long o = plane * zz;
      cp_async8(sv, usrc0 + o);
      if (has1) cp_async8(sv + 8u * T::NT, usrc1 + o);
    } else {
      const double* vp = vplane(g, h, U, zz);
      cp_async8(sv, vp + voff0);
      if (has1) cp_async8(sv + 8u * T::NT, vp + voff1);
    }
    if (zz >= zb && zz < ze) {
      const unsigned sc = sc0 + 8u * 4 * T::NT * ((zz - zb) & (kRG - 1));
      const long long i = ip + plane * zz;
      if (!d1_is_u) cp_async8(sc, a.d1 + i);
      if (has2) cp_async8(sc + 8u * T::NT, a.um2 + i);
      if (LAST) {
        cp_async8(sc + 16u * T::NT, a.g1v + i);
        if (!FIRST) cp_async8(sc + 24u * T::NT, a.g2v + i);
      }
    }
    cp_commit();
  };
  load_plane(zb - 1);
  load_plane(zb);
  load_plane(zb + 1);
  __syncthreads();  // publishes `skip`
  const bool skipped = skip != 0;
  bool bad_in = false, bad_out = false, guard = false;
  const int cell = (DIM == 3 ? (ty + 1) * T::HX : 0) + tx + 1;
  for (int z = zb; z < ze && !skipped; ++z) {
    if (z + 2 <= ze) load_plane(z + 2);
    else cp_commit();
    cp_wait<1>();
    __syncthreads();
    const int p = z - zb + 1;
    const double* V0 = vst + (p & (kRV - 1)) * T::VT;
    const double vc = V0[cell];
    double D = fma(g.wc, vc, g.w[DIM - 1] * (vst[((p - 1) & (kRV - 1)) * T::VT + cell] +
                                             vst[((p + 1) & (kRV - 1)) * T::VT + cell]));
    if (DIM >= 2) D = fma(g.w[0], V0[cell - 1] + V0[cell + 1], D);
    if (DIM == 3) D = fma(g.w[1], V0[cell - T::HX] + V0[cell + T::HX], D);
    const double* C0 = cst + ((z - zb) & (kRG - 1)) * 4 * T::NT + t;
    const double base = has2 ? fma(a.nu, vc, a.kappa * C0[T::NT]) : a.nu * vc;
    const double d1 = d1_is_u ? vc : C0[0];
    const double dk = fma(a.mueta, fma(d1, a.inv_mue1, D), base);
    if (valid) {
      const long long i = ip + plane * z;
      bad_in |= !finite_hi(dk);
      double vput = dk;
      if (!LAST) {
        a.uk[i] = dk;
      } else {
        const double gv = C0[2 * T::NT];
        const double b0 = FIRST ? gv : fma(a.onu, gv, a.okappa * C0[3 * T::NT]);
        const double o0 = fma(a.cG, dk, b0);
        a.outv[i] = o0;
        bad_out |= !finite_hi(o0);
        guard |= !(fabs(o0) <= 1e6);  // also a non-finite V
        vput = o0;
      }
      if (z == 0 && h.put_lo) h.put_lo[ip] = vput;
      if (z == g.nzl - 1 && h.put_hi) h.put_hi[ip] = vput;
    }
  }
  cp_wait<0>();
  halo_signal(h, zb == 0, ze >= g.nzl);
  if (skipped) return;
  const unsigned long long base = a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1));
  if (bad_in) atomicMin(a.event, base + a.k);
  if (LAST && bad_out) atomicMin(a.event, base + a.m + 1);
  if (LAST && a.last && guard)
    atomicMin(a.event, a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
}

// ---------------------------------------------------------------------------
// k_node_tma / k_vin_tma: the staged kernels with TMA. Thread 0 issues each
// plane's bulk tensor copies (V tile + halo, the tile's gates, g_{j-2})
// two planes ahead; they complete on the plane's mbarrier (transaction
// bytes), so the compute threads spend no instructions on loading. Halo
// cells past the grid edge arrive zero-filled: the compute reads the
// mirrored neighbour there instead (P/src/monodomain.cpp:85-86).
// ---------------------------------------------------------------------------
// The box's innermost start coordinate must be 16-byte aligned, so the V
// box spans x0-2 .. x0+TX+1 (two cells of halo on each side in x).
// Planes in flight ahead of the computed one. Ring limits: V stages need
// kTmaLA + 2 <= kRV; gate stages are refilled kTmaLA - 1 planes after their
// last read (one __syncthreads per plane), so kTmaLA <= kRG.
#ifndef EMRKC_TMA_LA
#define EMRKC_TMA_LA 3
#endif
constexpr int kTmaLA = EMRKC_TMA_LA;
#ifndef EMRKC_ISSUE1
#define EMRKC_ISSUE1 1
#endif
static_assert(kTmaLA >= 1 && kTmaLA + 2 <= kRV && kTmaLA <= kRG, "TMA lookahead");

template <int DIM>
struct TmaTile {
  using T = PipeTile<DIM>;
  static constexpr int HX = T::TX + 4;
  static constexpr int VT = HX * T::HY;           // V cells per stage
  static constexpr int VS = (VT + 15) & ~15;      // V stage stride (128-byte aligned)
};

// k_node_tma gate ring and barrier period: with FIRST (no g_{j-2} fields)
// the gate ring is deep enough for one __syncthreads per EMRKC_SYNCP planes
// (a slot is rewritten kRGn(FIRST) - kTmaLA planes after its last read).
#ifndef EMRKC_EVWARP1
#define EMRKC_EVWARP1 1
#endif
#ifndef EMRKC_SYNCP
#define EMRKC_SYNCP 1
#endif
template <int FIRST>
__host__ __device__ constexpr int kRGn() { return FIRST && EMRKC_SYNCP > 1 ? 8 : kRG; }
template <int FIRST>
__host__ __device__ constexpr int kSyncP() { return FIRST ? EMRKC_SYNCP : 1; }
static_assert(EMRKC_SYNCP == 1 || (EMRKC_SYNCP == 2 && kTmaLA + 4 <= kRV),
              "k_node_tma barrier period");

template <int DIM, int FIRST>
constexpr size_t tma_node_smem_bytes(int naux = 0) {
  using T = PipeTile<DIM>;
  return sizeof(double) * (kRV * TmaTile<DIM>::VS + kRGn<FIRST>() * (3 + naux) * T::NT +
                           (FIRST ? 0 : kRG * (4 + naux) * T::NT)) + 128;
}

// Issues the V box of local plane zz (interior, mirror, or ghost).
template <int DIM>
__device__ __forceinline__ void tma_vplane(const Geom& g, const CUtensorMap* vmap,
                                           const CUtensorMap* glo, const CUtensorMap* ghi,
                                           bool has_lo, bool has_hi, unsigned dst,
                                           unsigned bar, int x0, int y0, int zz) {
  int lz = zz;
  if (zz < 0 || zz >= g.nzl) {
    int gz = zz + g.zoff;
    gz = gz < 0 ? 1 : (gz >= g.nzg ? g.nzg - 2 : gz);
    lz = gz - g.zoff;
  }
  if (lz >= 0 && lz < g.nzl) {
    if (DIM == 3) tma_load_3d(dst, vmap, bar, x0 - 2, y0 - 1, lz);
    else tma_load_2d(dst, vmap, bar, x0 - 2, lz);
  } else {
    const CUtensorMap* gm = lz < 0 ? glo : ghi;
    if (DIM == 3) tma_load_2d(dst, gm, bar, x0 - 2, y0 - 1);
    else tma_load_1d(dst, gm, bar, x0 - 2);
  }
  (void)has_lo;
  (void)has_hi;
}

// AUX = 0 compiles the aux rows out (HH proper: constant ring strides, no
// per-plane aux loop); AUX = 1 is the synthetic width stand-in (g.naux > 0).
template <int DIM, int FIRST, int ION, int AUX>
__global__ void __launch_bounds__(PipeTile<DIM>::NT, EMRKC_PIPE_MINBLOCKS)
    k_node_tma(const Geom g, const Halo h, const FastArgs a, const __grid_constant__ TmaNode tm) {
  using T = PipeTile<DIM>;
  constexpr int VS = TmaTile<DIM>::VS;
  extern __shared__ __align__(128) double smem_tma[];
  // 128-byte aligned stage base (pointer arithmetic keeps the shared space)
  double* vst = smem_tma + ((128u - (smem_u32(smem_tma) & 127u)) & 127u) / 8;  // [kRV][VS]
  // gate stage: the three gates and the aux fields of the synthetic width
  // stand-in (g.naux, include/emrkc.h), fields 1 .. nf - 1 of g_{j-1}
  const int NA = AUX ? g.naux : 0;
  const int GF = 3 + NA, QF = 4 + NA;
  double* gst = vst + kRV * VS;                     // [kRG][GF][NT]
  constexpr int RG = kRGn<FIRST>();
  double* g2s = gst + RG * GF * T::NT;              // [kRG][QF][NT]
  __shared__ double tab[256];
  __shared__ __align__(8) unsigned long long bars[kRV];
  __shared__ int skip;
  const int t = threadIdx.x;
  const int zb = a.z_lo + (DIM == 3 ? blockIdx.z : blockIdx.y) * a.zc;
  const int ze = min(a.z_hi, zb + a.zc);
  pdl_launch_dependents();
  if (t == 0) {  // prologue that reads nothing the previous kernel writes
    for (int s = 0; s < kRV; ++s) mbar_init(smem_u32(&bars[s]), 1);
    mbar_fence_init();
    prefetch_tensormap(&tm.v);
    prefetch_tensormap(&tm.gates);
    if (!FIRST) prefetch_tensormap(&tm.g2);
  }
  __syncthreads();  // barriers initialised before any warp issues onto them
  const int tx = t % T::TX, ty = t / T::TX;
  const int x0 = blockIdx.x * T::TX;
  const int y0 = DIM == 3 ? blockIdx.y * T::TY : 0;
  const int cx = x0 + tx, cy = y0 + ty;
  const bool valid = cx < g.n0 && (DIM == 2 || cy < g.n1);
  const long long ip = valid ? (long long)cx + (long long)g.n0 * cy : 0;
  const long long nn = g.nn, plane = g.plane;
  const unsigned v0 = smem_u32(vst), gs0 = smem_u32(gst), qs0 = smem_u32(g2s);
  const unsigned b0 = smem_u32(bars);
  constexpr unsigned vbytes = 8u * TmaTile<DIM>::VT;
  const unsigned cbytes = 8u * T::NT * (GF + (FIRST ? 0 : QF));
  // The copies of a plane are issued by lane 0 of warps 0 (expect_tx + V
  // box), 1 (gate box) and 2 (g_{j-2} box): the issue work is spread over
  // three warps instead of serialising one before the per-plane barrier.
  const int role = (t & 31) == 0 ? (t >> 5) : -1;
  auto issue_comp = [&](int zz) {  // plane zz in [zb, ze)
    const int q = zz - zb + 1;
    const unsigned bar = b0 + 8u * (q & (kRV - 1));
    const unsigned sg = (unsigned)((zz - zb) & (RG - 1));
    if (role == 0) {
      mbar_expect_tx(bar, vbytes + cbytes);
      const unsigned vd = v0 + 8u * VS * (q & (kRV - 1));
      if (DIM == 3) tma_load_3d(vd, &tm.v, bar, x0 - 2, y0 - 1, zz);
      else tma_load_2d(vd, &tm.v, bar, x0 - 2, zz);
    }
    if (role == (EMRKC_ISSUE1 ? 0 : 1)) {
      if (DIM == 3) tma_load_4d(gs0 + 8u * GF * T::NT * sg, &tm.gates, bar, x0, y0, zz, 1);
      else tma_load_3d(gs0 + 8u * GF * T::NT * sg, &tm.gates, bar, x0, zz, 1);
    }
    if (!FIRST && role == (EMRKC_ISSUE1 ? 0 : 2)) {
      if (DIM == 3) tma_load_4d(qs0 + 8u * QF * T::NT * sg, &tm.g2, bar, x0, y0, zz, 0);
      else tma_load_3d(qs0 + 8u * QF * T::NT * sg, &tm.g2, bar, x0, zz, 0);
    }
  };
  // halo plane zb - 1 or ze (V only; mirror or ghost at the slab edge)
  auto issue_edge = [&](int zz, unsigned extra) {
    if (role != 0) return;
    const int q = zz - zb + 1;
    const unsigned bar = b0 + 8u * (q & (kRV - 1));
    mbar_expect_tx(bar, vbytes + extra);
    tma_vplane<DIM>(g, &tm.v, &tm.glo, &tm.ghi, h.lo != nullptr, h.hi != nullptr,
                    v0 + 8u * VS * (q & (kRV - 1)), bar, x0, y0, zz);
  };
  pdl_wait();
  halo_wait(h, zb == 0, ze >= g.nzl);
  int nq = 0;  // prologue loads (planes zb - 1 ...)
  if (EMRKC_ISSUE1 ? role == 0 : (role >= 0 && role <= 2)) {
    if (role == 0) {
      // ghost planes arrived through generic peer stores (acquired in
      // halo_wait); order them before this thread's async-proxy reads
      fence_proxy_async();
      bulk_load(smem_u32(tab), kExp2Tab256, sizeof(double) * 256, b0);  // exp table
    }
    issue_edge(zb - 1, sizeof(double) * 256);
    nq = 1;
    for (int i = 0; i < kTmaLA; ++i, ++nq) {
      if (zb + i < ze) issue_comp(zb + i);
      else {
        issue_edge(ze, 0);
        ++nq;
        break;
      }
    }
  }
  if (t == (EMRKC_EVWARP1 ? 32 : 0)) skip = (*(volatile const unsigned long long*)a.event) < level_floor(a.code_base, a.j, a.m, 1);
  __syncthreads();
  const bool skipped = skip != 0;
  if (skipped) {  // aborted earlier: drain the prologue copies, release the neighbours
    const int np = 1 + min(kTmaLA, ze - zb) + (ze - zb < kTmaLA ? 1 : 0);
    for (int q = 0; q < np; ++q) mbar_wait(b0 + 8u * q, 0);
    put_signal(h, put_plan(h, g.nzl), zb, ze);
    return;
  }
  (void)nq;
  // mirrored in-plane neighbours at the grid edge (halo cells there are 0)
  constexpr int HXT = TmaTile<DIM>::HX;
  const int cell = (DIM == 3 ? (ty + 1) * HXT : 0) + tx + 2;
  const int cxm = cell + (cx > 0 ? -1 : 1), cxp = cell + (cx < g.n0 - 1 ? 1 : -1);
  const int cym = cell + (cy > 0 ? -HXT : HXT), cyp = cell + (cy < g.n1 - 1 ? HXT : -HXT);
  int zs0 = 1, zs1 = 0;
  if (valid && stim_col_xy<DIM>(g, cx, cy)) {
    zs0 = g.st_lo[DIM - 1] - g.zoff;
    zs1 = g.st_hi[DIM - 1] - g.zoff;
  }
  bool bad = false, guard = false;
  // finite test folded over the hot loop: min over nodes of the sum's
  // (~hi & exponent mask); 0 means some node produced Inf/NaN
  unsigned finacc = 0x7ff00000u;
  unsigned long long slow_mask = 0;  // planes z - zb (< kMaxZc = 64) left to the reference path
  double glo = 2.0, ghi = -1.0;
  double* po = a.out + ip + plane * zb;
  double* pu = ION ? a.u1 + ip + plane * zb : nullptr;
  if (!skipped) {
    mbar_wait(b0, 0);       // plane zb - 1
    mbar_wait(b0 + 8u, 0);  // plane zb
  }
  // halo puts hoisted: planes z < pp.zl / z >= pp.zh of this column go to
  // the neighbours' ghosts (one plane, or K planes of d_1 for the wide halo)
  const PutPlan pp = put_plan(h, g.nzl);
  for (int z = zb; z < ze && !skipped; ++z) {
    const int p = z - zb + 1;
    if (EMRKC_ISSUE1 ? role == 0 : role >= 0) {
      if (z + kTmaLA < ze) issue_comp(z + kTmaLA);
      else if (z + kTmaLA == ze) issue_edge(ze, 0);
    }
    mbar_wait(b0 + 8u * ((p + 1) & (kRV - 1)), ((p + 1) >> 3) & 1);
    const double* V0 = vst + (p & (kRV - 1)) * VS;
    const double vc = V0[cell];
    const double vm = vst[((p - 1) & (kRV - 1)) * VS + cell];
    const double vp = vst[((p + 1) & (kRV - 1)) * VS + cell];
    double xs = 0.0, ys = 0.0;
    if (DIM >= 2) xs = V0[cxm] + V0[cxp];
    if (DIM == 3) ys = V0[cym] + V0[cyp];
    const double* G0 = gst + ((z - zb) & (RG - 1)) * GF * T::NT + t;
    const double* Q0 = g2s + ((z - zb) & (RG - 1)) * QF * T::NT + t;
    const double z0 = G0[0], z1 = G0[T::NT], z2 = G0[2 * T::NT];
    const bool fast = fabs(vc - a.vmid) <= a.vfast;
    if (!fast) slow_mask |= 1ull << (z - zb);
    NodeOut r = node_update_s<DIM, FIRST, ION, 0>(
        g, a, tab, vm, vc, vp, xs, ys, z0, z1, z2, 0.0,
        Q0, T::NT);
    if (z >= zs0 && z <= zs1) {
      if (ION) r.o0 = fma(a.mue1, a.stim, r.o0);
      else r.o0 = fma(a.cV, a.stim, r.o0);
    }
    if (valid && fast) {
      po[nn] = r.o1;
      po[2 * nn] = r.o2;
      po[3 * nn] = r.o3;
      if (ION) {
        *pu = r.o0;
      } else {
        *po = r.o0;
        guard |= !(fabs(r.o0) <= 1e6);  // also a non-finite V
      }
      finacc = min(finacc, ~(unsigned)__double2hiint((r.o0 + r.o1) + (r.o2 + r.o3)) & 0x7ff00000u);
      // aux rows: y_E = z (no exponential part), f_S = g_S(V, z), the inner
      // iterate z + c_m eta g_S, g_j = base + (mu_j dt c_m) g_S
      for (int q = 0; q < NA; ++q) {
        const double za = G0[(3 + q) * T::NT];
        const double base = FIRST ? za : fma(a.nu, za, a.kappa * Q0[(4 + q) * T::NT]);
        const double oa = fma(a.cA, aux_rate_fast(q, vc, za), base);
        po[(4 + q) * nn] = oa;
        finacc = min(finacc, ~(unsigned)__double2hiint(oa) & 0x7ff00000u);
      }
      if (z < pp.zl) pp.plo[ip + plane * z] = r.o0;
      if (z >= pp.zh) pp.phi[ip + plane * (z - pp.zh)] = r.o0;
      if (a.last) {  // std::min / std::max per value (NaN skipped), select form
        glo = r.o1 < glo ? r.o1 : glo;
        ghi = ghi < r.o1 ? r.o1 : ghi;
        glo = r.o2 < glo ? r.o2 : glo;
        ghi = ghi < r.o2 ? r.o2 : ghi;
        glo = r.o3 < glo ? r.o3 : glo;
        ghi = ghi < r.o3 ? r.o3 : ghi;
      }
    }
    po += plane;
    if (ION) pu += plane;
    // stage (p - 5) may be refilled next iteration; with a period of 2 the
    // deeper gate ring keeps every refill behind a barrier
    if (kSyncP<FIRST>() == 1 || ((z - zb) & 1)) __syncthreads();
  }
  bad = finacc == 0u;
  if (!skipped && valid && slow_mask) {
    const Nbr<DIM> o = nbr_of<DIM>(g, Col<DIM>{cx, cy, ip, zb, ze, true});
    const double* G = a.g1;
    for (int z = zb; z < ze; ++z) {
      if (!(slow_mask >> (z - zb) & 1ull)) continue;
      const long long i = ip + plane * z;
      const double vc = __ldg(G + i);
      const double vm = zval(G, g, ip, z - 1, h.lo, h.hi);
      const double vp = zval(G, g, ip, z + 1, h.lo, h.hi);
      double xs = 0.0, ys = 0.0;
      if (DIM >= 2) xs = __ldg(G + i + o.xm) + __ldg(G + i + o.xp);
      if (DIM == 3) ys = __ldg(G + i + o.ym) + __ldg(G + i + o.yp);
      const double stim = (z >= zs0 && z <= zs1) ? a.stim : 0.0;
      double q[4] = {0.0, 0.0, 0.0, 0.0};
      if (!FIRST)
        for (int f = 0; f < 4; ++f) q[f] = __ldg(a.g2 + f * nn + i);
      const NodeOut r = node_update_s<DIM, FIRST, ION, 1>(
          g, a, tab, vm, vc, vp, xs, ys, __ldg(G + nn + i), __ldg(G + 2 * nn + i),
          __ldg(G + 3 * nn + i), stim, q, 1);
      a.out[nn + i] = r.o1;
      a.out[2 * nn + i] = r.o2;
      a.out[3 * nn + i] = r.o3;
      if (ION) {
        a.u1[i] = r.o0;
      } else {
        a.out[i] = r.o0;
        guard |= !(fabs(r.o0) <= 1e6);  // also a non-finite V
      }
      bad |= !finite_hi((r.o0 + r.o1) + (r.o2 + r.o3));
      for (int q = 0; q < NA; ++q) {
        const double za = __ldg(G + (4 + q) * nn + i);
        const double base = FIRST ? za : fma(a.nu, za, a.kappa * __ldg(a.g2 + (4 + q) * nn + i));
        const double oa = fma(a.cA, aux_rate_fast(q, vc, za), base);
        a.out[(4 + q) * nn + i] = oa;
        bad |= !finite_hi(oa);
      }
      if (z < pp.zl) pp.plo[ip + plane * z] = r.o0;
      if (z >= pp.zh) pp.phi[ip + plane * (z - pp.zh)] = r.o0;
      if (a.last) {
        glo = fmin(glo, fmin(r.o1, fmin(r.o2, r.o3)));
        ghi = fmax(ghi, fmax(r.o1, fmax(r.o2, r.o3)));
      }
    }
  }
  put_signal(h, pp, zb, ze);
  if (skipped) return;
  if (bad && !a.exex) {  // EXEX-RL never throws NumericalAbort
    Col<DIM> c;
    c.c0 = cx;
    c.c1 = cy;
    c.ip = ip;
    c.z0 = zb;
    c.z1 = ze;
    c.valid = true;
    const bool inner = inner_nonfinite<DIM>(g, h, a.g1, c, nbr_of<DIM>(g, c), a.eta);
    atomicMin(a.event, a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1)) +
                           (inner ? 1 : a.m + 1));
  }
  if (!ION && a.last && guard)
    atomicMin(a.event, a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
  if (a.last) block_gate_range_d(a.gate_slot, glo, ghi, valid && ze > zb);
}

// ---------------------------------------------------------------------------
// k_node_pair<FIRST, ION>: k_node_tma's outer stage (3-D, HH proper, whole
// grid) with an x-adjacent PAIR of nodes per thread: 64 x 4 tiles, 128
// threads. k_node_tma spends ~140 of its ~340 warp instructions per node on
// per-plane work that does not depend on the node count (ring and address
// arithmetic, barrier, mbarrier wait, parameter loads, stimulus / range
// tests); here that work serves two nodes, and
//   * the z neighbours of a column are the thread's own registers (a
//     (z - 1, z) window; one 128-bit shared load brings plane z + 1 of both
//     nodes), the inner x neighbours are the pair's own values: 5 shared
//     loads of V per pair (3 x 128 bit, 2 x 64 bit) instead of 14;
//   * gates arrive with one 128-bit shared load per field and every output
//     field leaves with one 128-bit global store per pair;
//   * finite tests run on the integer pipe (max over hi | 0x800fffff).
// Same node arithmetic (node_update_s) in the same order: bitwise equal to
// k_node_tma (tests/test_gpu_kernel_families.py). No slab faces: partitioned
// handles, aux rows and 2-D grids keep k_node_tma.
// ---------------------------------------------------------------------------
constexpr int kPairTX = 64, kPairTY = 4, kPairNT = 128;
constexpr int kPairHX = kPairTX + 4, kPairHY = kPairTY + 2;  // V box 68 x 6 (x0 - 2, y0 - 1)
constexpr int kPairVT = kPairHX * kPairHY;
constexpr int kPairVS = (kPairVT + 15) & ~15;
constexpr int kPairCS = kPairTX * kPairTY;  // cells of one centre field

// Tile shapes of k_node_pair: 64 x 4 (a warp per row) or 32 x 8 (half a warp
// per row) for grids whose width wastes fewer lanes in 32-wide tiles
// (n0 = 200: 224 / 200 against 256 / 200 columns).
template <int TXW>
struct PairTile {
  static constexpr int TX = TXW, TY = kPairNT * 2 / TXW, PPR = TXW / 2;  // pairs per row
  static constexpr int HX = TX + 4, HY = TY + 2;                         // V box (x0 - 2, y0 - 1)
  static constexpr int VT = HX * HY, VS = (VT + 15) & ~15, CS = TX * TY;
};
template <int FIRST, int TXW>
constexpr size_t pair_smem_bytes() {
  using P = PairTile<TXW>;
  return sizeof(double) * (kRV * P::VS + kRG * 3 * P::CS + (FIRST ? 0 : kRG * 4 * P::CS)) + 128;
}

__device__ __forceinline__ unsigned nf_hi(double v) {
  return (unsigned)__double2hiint(v) | 0x800fffffu;
}

template <int FIRST, int ION, int TXW>
__global__ void __launch_bounds__(kPairNT, FIRST ? 4 : 2)
    k_node_pair(const Geom g, const Halo h, const FastArgs a, const __grid_constant__ TmaNode tm) {
  using P = PairTile<TXW>;
  constexpr int VS = P::VS, CS = P::CS, HXT = P::HX;
  extern __shared__ __align__(128) double smem_tma[];
  double* vst = smem_tma + ((128u - (smem_u32(smem_tma) & 127u)) & 127u) / 8;  // [kRV][VS]
  double* gst = vst + kRV * VS;        // [kRG][3][CS]
  double* g2s = gst + kRG * 3 * CS;    // [kRG][4][CS]
  __shared__ double tab[256];
  __shared__ __align__(8) unsigned long long bars[kRV];
  __shared__ int skip;
  const int t = threadIdx.x;
  const int zb = a.z_lo + blockIdx.z * a.zc;
  const int ze = min(a.z_hi, zb + a.zc);
  pdl_launch_dependents();
  if (t == 0) {  // prologue that reads nothing the previous kernel writes
    for (int s = 0; s < kRV; ++s) mbar_init(smem_u32(&bars[s]), 1);
    mbar_fence_init();
    prefetch_tensormap(&tm.v);
    prefetch_tensormap(&tm.gates);
    if (!FIRST) prefetch_tensormap(&tm.g2);
  }
  __syncthreads();
  const int px = t % P::PPR, ty = t / P::PPR;
  const int x0 = blockIdx.x * P::TX, y0 = blockIdx.y * P::TY;
  const int cx = x0 + 2 * px, cy = y0 + ty;  // cell 0; cell 1 = (cx + 1, cy)
  const bool valid = cx < g.n0 && cy < g.n1;  // n0 is even: both cells or none
  const long long ip = valid ? (long long)cx + (long long)g.n0 * cy : 0;
  const long long nn = g.nn, plane = g.plane;
  const unsigned v0 = smem_u32(vst), gs0 = smem_u32(gst), qs0 = smem_u32(g2s);
  const unsigned b0 = smem_u32(bars);
  constexpr unsigned vbytes = 8u * P::VT;
  constexpr unsigned cbytes = 8u * CS * (3 + (FIRST ? 0 : 4));
  auto issue_comp = [&](int zz) {  // thread 0: plane zz in [zb, ze)
    const int q = zz - zb + 1;
    const unsigned bar = b0 + 8u * (q & (kRV - 1));
    const unsigned sg = (unsigned)((zz - zb) & (kRG - 1));
    mbar_expect_tx(bar, vbytes + cbytes);
    tma_load_3d(v0 + 8u * VS * (q & (kRV - 1)), &tm.v, bar, x0 - 2, y0 - 1, zz);
    tma_load_4d(gs0 + 8u * 3 * CS * sg, &tm.gates, bar, x0, y0, zz, 1);
    if (!FIRST) tma_load_4d(qs0 + 8u * 4 * CS * sg, &tm.g2, bar, x0, y0, zz, 0);
  };
  // halo plane zb - 1 or ze (V only; mirror or ghost at the slab edge)
  auto issue_edge = [&](int zz, unsigned extra) {
    const int q = zz - zb + 1;
    const unsigned bar = b0 + 8u * (q & (kRV - 1));
    mbar_expect_tx(bar, vbytes + extra);
    tma_vplane<3>(g, &tm.v, &tm.glo, &tm.ghi, h.lo != nullptr, h.hi != nullptr,
                  v0 + 8u * VS * (q & (kRV - 1)), bar, x0, y0, zz);
  };
  // a block stands for its 32-wide tiles in the neighbours' arrival counts
  // (halo_signals_pipe counts 32 x 4 tiles whatever kernel stores the planes)
  const int sigw = (P::TX > kTX3 ? 1 + (x0 + kTX3 < g.n0 ? 1 : 0) : 1) *
                   (P::TY > kTY3 ? 1 + (y0 + kTY3 < g.n1 ? 1 : 0) : 1);
  pdl_wait();
  halo_wait(h, zb == 0, ze >= g.nzl);
  if (t == 0) {
    // ghost planes arrived through generic peer stores (acquired in
    // halo_wait); order them before this thread's async-proxy reads
    fence_proxy_async();
    bulk_load(smem_u32(tab), kExp2Tab256, sizeof(double) * 256, b0);  // exp table
    issue_edge(zb - 1, sizeof(double) * 256);
    for (int i = 0; i < kTmaLA; ++i) {
      if (zb + i < ze) issue_comp(zb + i);
      else {
        issue_edge(ze, 0);
        break;
      }
    }
  }
  if (t == 32) skip = (*(volatile const unsigned long long*)a.event) < level_floor(a.code_base, a.j, a.m, 1);
  __syncthreads();
  if (skip != 0) {  // aborted earlier: drain the prologue copies
    const int np = 1 + min(kTmaLA, ze - zb) + (ze - zb < kTmaLA ? 1 : 0);
    for (int q = 0; q < np; ++q) mbar_wait(b0 + 8u * q, 0);
    const PutPlan pq = put_plan(h, g.nzl);  // release the neighbours
    halo_signal_w(h, sigw * max(0, min(ze, pq.zl) - zb), sigw * max(0, ze - max(zb, pq.zh)));
    return;
  }
  // cell 0 of the pair in a V stage; mirrored in-plane neighbours at the
  // grid edge (halo cells there are 0): x - 1 of cell 0, x + 1 of cell 1
  const int cell = (ty + 1) * HXT + 2 * px + 2;
  const int cxm = cell + (cx > 0 ? -1 : 1), cxp = cell + 1 + (cx + 1 < g.n0 - 1 ? 1 : -1);
  const int cym = cell + (cy > 0 ? -HXT : HXT), cyp = cell + (cy < g.n1 - 1 ? HXT : -HXT);
  const int gcell = ty * P::TX + 2 * px;  // the pair in a centre field
  int zs0 = 1, zs1 = 0;
  const bool st0 = valid && stim_col_xy<3>(g, cx, cy), st1 = valid && stim_col_xy<3>(g, cx + 1, cy);
  if (st0 || st1) {
    zs0 = g.st_lo[2] - g.zoff;
    zs1 = g.st_hi[2] - g.zoff;
  }
  bool guard = false;
  // Gate range of the step (P/src/simulate.cpp:76-85). With the range of
  // everything before this step (a.gate_prev: positive finite bounds) a value
  // whose high word lies strictly between the bounds' high words cannot
  // extend the run's range: those skip the FP64 min / max (integer pipe
  // test per pair); negative and non-finite values always take the exact path.
  double glo = 2.0, ghi = -1.0;
  unsigned tlo = 0xffffffffu, thi = 0u;  // exact path iff hmin <= tlo || hmax >= thi
  unsigned long long plo = ~0ull, phi = 0ull;
  if (a.last && a.gate_prev) {
    plo = a.gate_prev[0];
    phi = a.gate_prev[1];
    const unsigned hl = (unsigned)((plo ^ 0x8000000000000000ull) >> 32);
    const unsigned hh = (unsigned)((phi ^ 0x8000000000000000ull) >> 32);
    if (plo != ~0ull && (plo >> 63) && (phi >> 63) && hh < 0x7ff00000u && hl <= hh) {
      tlo = hl;
      thi = hh;
      // the running min / max start from the earlier range (no sentinels)
      glo = __longlong_as_double((long long)(plo ^ 0x8000000000000000ull));
      ghi = __longlong_as_double((long long)(phi ^ 0x8000000000000000ull));
    } else {
      plo = ~0ull;
      phi = 0ull;
    }
  }
  unsigned nfacc = 0u;  // all ones once an output was non-finite
  unsigned long long slow_mask = 0;  // planes z - zb (< kMaxZc = 64) left to the reference path
  double* po = a.out + ip + plane * zb;
  double* pu = ION ? a.u1 + ip + plane * zb : nullptr;
  mbar_wait(b0, 0);       // plane zb - 1
  mbar_wait(b0 + 8u, 0);  // plane zb
  // z window of the two columns: planes z - 1 and z
  double2 wm = *reinterpret_cast<const double2*>(vst + cell);
  double2 wc = *reinterpret_cast<const double2*>(vst + VS + cell);
  // halo puts: planes z < pp.zl / z >= pp.zh of this column go to the
  // neighbours' ghosts (one plane, or K planes of d_1 for the wide halo)
  const PutPlan pp = put_plan(h, g.nzl);
  for (int z = zb; z < ze; ++z) {
    const int p = z - zb + 1;
    if (t == 0) {
      if (z + kTmaLA < ze) issue_comp(z + kTmaLA);
      else if (z + kTmaLA == ze) issue_edge(ze, 0);
    }
    mbar_wait(b0 + 8u * ((p + 1) & (kRV - 1)), ((p + 1) >> 3) & 1);
    const double* V0 = vst + (p & (kRV - 1)) * VS;
    const double2 wp = *reinterpret_cast<const double2*>(vst + ((p + 1) & (kRV - 1)) * VS + cell);
    const double2 ym = *reinterpret_cast<const double2*>(V0 + cym);
    const double2 yp = *reinterpret_cast<const double2*>(V0 + cyp);
    const double xm0 = V0[cxm], xp1 = V0[cxp];
    const double* G0 = gst + ((z - zb) & (kRG - 1)) * 3 * CS + gcell;
    const double* Q0 = g2s + ((z - zb) & (kRG - 1)) * 4 * CS + gcell;
    const double2 za = *reinterpret_cast<const double2*>(G0);
    const double2 zb2 = *reinterpret_cast<const double2*>(G0 + CS);
    const double2 zc2 = *reinterpret_cast<const double2*>(G0 + 2 * CS);
    // window test on the integer pipe (conservative; the per-node path below
    // applies the exact test to the planes it defers)
    const int hx = __double2hiint(wc.x), hy = __double2hiint(wc.y);
    const bool fast = hx < a.vq_pos && (unsigned)hx < a.vq_neg && hy < a.vq_pos &&
                      (unsigned)hy < a.vq_neg;
    if (!fast) slow_mask |= 1ull << (z - zb);
    NodeOut r0 = node_update_s<3, FIRST, ION, 0>(g, a, tab, wm.x, wc.x, wp.x, xm0 + wc.y,
                                                 ym.x + yp.x, za.x, zb2.x, zc2.x, 0.0, Q0, CS);
    NodeOut r1 = node_update_s<3, FIRST, ION, 0>(g, a, tab, wm.y, wc.y, wp.y, wc.x + xp1,
                                                 ym.y + yp.y, za.y, zb2.y, zc2.y, 0.0, Q0 + 1, CS);
    if (z >= zs0 && z <= zs1) {
      const double sc = ION ? a.mue1 : a.cV;
      if (st0) r0.o0 = fma(sc, a.stim, r0.o0);
      if (st1) r1.o0 = fma(sc, a.stim, r1.o0);
    }
    if (valid && fast) {
      *reinterpret_cast<double2*>(po + nn) = make_double2(r0.o1, r1.o1);
      *reinterpret_cast<double2*>(po + 2 * nn) = make_double2(r0.o2, r1.o2);
      *reinterpret_cast<double2*>(po + 3 * nn) = make_double2(r0.o3, r1.o3);
      if (ION) {
        *reinterpret_cast<double2*>(pu) = make_double2(r0.o0, r1.o0);
      } else {
        *reinterpret_cast<double2*>(po) = make_double2(r0.o0, r1.o0);
        guard |= !(fabs(r0.o0) <= 1e6) || !(fabs(r1.o0) <= 1e6);  // also a non-finite V
      }
      if (z < pp.zl) *reinterpret_cast<double2*>(pp.plo + ip + plane * z) = make_double2(r0.o0, r1.o0);
      if (z >= pp.zh)
        *reinterpret_cast<double2*>(pp.phi + ip + plane * (z - pp.zh)) = make_double2(r0.o0, r1.o0);
      nfacc = max(max(nfacc, max(nf_hi(r0.o0), nf_hi(r0.o1))), max(nf_hi(r0.o2), nf_hi(r0.o3)));
      nfacc = max(max(nfacc, max(nf_hi(r1.o0), nf_hi(r1.o1))), max(nf_hi(r1.o2), nf_hi(r1.o3)));
      bool track = a.last;
      if (track) {
        const unsigned h0 = __double2hiint(r0.o1), h1 = __double2hiint(r0.o2),
                       h2 = __double2hiint(r0.o3), h3 = __double2hiint(r1.o1),
                       h4 = __double2hiint(r1.o2), h5 = __double2hiint(r1.o3);
        const unsigned hmin = min(min(min(h0, h1), min(h2, h3)), min(h4, h5));
        const unsigned hmax = max(max(max(h0, h1), max(h2, h3)), max(h4, h5));
        track = hmin <= tlo || hmax >= thi;
      }
      if (track) {  // std::min / std::max per value (NaN skipped), select form
        glo = r0.o1 < glo ? r0.o1 : glo;
        ghi = ghi < r0.o1 ? r0.o1 : ghi;
        glo = r0.o2 < glo ? r0.o2 : glo;
        ghi = ghi < r0.o2 ? r0.o2 : ghi;
        glo = r0.o3 < glo ? r0.o3 : glo;
        ghi = ghi < r0.o3 ? r0.o3 : ghi;
        glo = r1.o1 < glo ? r1.o1 : glo;
        ghi = ghi < r1.o1 ? r1.o1 : ghi;
        glo = r1.o2 < glo ? r1.o2 : glo;
        ghi = ghi < r1.o2 ? r1.o2 : ghi;
        glo = r1.o3 < glo ? r1.o3 : glo;
        ghi = ghi < r1.o3 ? r1.o3 : ghi;
      }
    }
    wm = wc;
    wc = wp;
    po += plane;
    if (ION) pu += plane;
    __syncthreads();  // stage (p - 5) may be refilled next iteration
  }
  bool bad = nfacc == 0xffffffffu;
  if (valid && slow_mask) {  // planes with a node outside the fast window: reference-order path
    for (int c = 0; c < 2; ++c) {
      const long long ipc = ip + c;
      const Nbr<3> o = nbr_of<3>(g, Col<3>{cx + c, cy, ipc, zb, ze, true});
      const double* G = a.g1;
      const bool stc = c ? st1 : st0;
      for (int z = zb; z < ze; ++z) {
        if (!(slow_mask >> (z - zb) & 1ull)) continue;
        const long long i = ipc + plane * z;
        const double vc = __ldg(G + i);
        const double vm = zval(G, g, ipc, z - 1, h.lo, h.hi);
        const double vp = zval(G, g, ipc, z + 1, h.lo, h.hi);
        const double xs = __ldg(G + i + o.xm) + __ldg(G + i + o.xp);
        const double ys = __ldg(G + i + o.ym) + __ldg(G + i + o.yp);
        const double stim = (stc && z >= zs0 && z <= zs1) ? a.stim : 0.0;
        double q[4] = {0.0, 0.0, 0.0, 0.0};
        if (!FIRST)
          for (int f = 0; f < 4; ++f) q[f] = __ldg(a.g2 + f * nn + i);
        // a node inside the window whose partner is not: the hot loop's form
        // (stimulus added to the result), so both kernels agree bit for bit
        NodeOut r;
        if (fabs(vc - a.vmid) <= a.vfast) {
          r = node_update_s<3, FIRST, ION, 0>(g, a, tab, vm, vc, vp, xs, ys, __ldg(G + nn + i),
                                              __ldg(G + 2 * nn + i), __ldg(G + 3 * nn + i), 0.0,
                                              q, 1);
          if (stc && z >= zs0 && z <= zs1) r.o0 = fma(ION ? a.mue1 : a.cV, a.stim, r.o0);
        } else {
          r = node_update_s<3, FIRST, ION, 1>(g, a, tab, vm, vc, vp, xs, ys, __ldg(G + nn + i),
                                              __ldg(G + 2 * nn + i), __ldg(G + 3 * nn + i), stim,
                                              q, 1);
        }
        a.out[nn + i] = r.o1;
        a.out[2 * nn + i] = r.o2;
        a.out[3 * nn + i] = r.o3;
        if (ION) {
          a.u1[i] = r.o0;
        } else {
          a.out[i] = r.o0;
          guard |= !(fabs(r.o0) <= 1e6);  // also a non-finite V
        }
        bad |= !finite_hi((r.o0 + r.o1) + (r.o2 + r.o3));
        if (z < pp.zl) pp.plo[ipc + plane * z] = r.o0;
        if (z >= pp.zh) pp.phi[ipc + plane * (z - pp.zh)] = r.o0;
        if (a.last) {
          glo = fmin(glo, fmin(r.o1, fmin(r.o2, r.o3)));
          ghi = fmax(ghi, fmax(r.o1, fmax(r.o2, r.o3)));
        }
      }
    }
  }
  halo_signal_w(h, sigw * max(0, min(ze, pp.zl) - zb), sigw * max(0, ze - max(zb, pp.zh)));
  if (bad && !a.exex) {  // EXEX-RL never throws NumericalAbort
    bool inner = false;
    for (int c = 0; c < 2; ++c) {
      Col<3> col;
      col.c0 = cx + c;
      col.c1 = cy;
      col.ip = ip + c;
      col.z0 = zb;
      col.z1 = ze;
      col.valid = true;
      inner |= inner_nonfinite<3>(g, h, a.g1, col, nbr_of<3>(g, col), a.eta);
    }
    atomicMin(a.event, a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1)) +
                           (inner ? 1 : a.m + 1));
  }
  if (!ION && a.last && guard)
    atomicMin(a.event, a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
  if (a.last) {
    // fold the earlier range in: the slot is cumulative when a.gate_prev is
    // used (values skipped above lie strictly inside it)
    unsigned long long lo = valid && ze > zb ? ord_of(glo) : ~0ull;
    unsigned long long hi = valid && ze > zb ? ord_of(ghi) : 0ull;
    block_gate_range(a.gate_slot, min(lo, plo), max(hi, phi));
  }
}

// ---------------------------------------------------------------------------
// k_step_x: cross-step fusion of the s = 1, m = 2 step (EMRKC_XSTEP=1, 3-D
// whole grids, HH proper). One launch does inner stage 2 of step n AND the
// node update (exponential Euler + inner stage 1) of step n + 1:
//   W = V_{n+1} = V_n + cG d_2,  d_2 = nu'_2 d_1 + mu'_2 eta (d_1 / (mu'_1 eta) + f_F(d_1))
// is a 12-flop stencil of the complete fields d_1^n and V_n, so a block
// computes it on its 64 x 4 tile plus a one-cell halo (the halo twice, by the
// neighbouring blocks too: no exchange between blocks) straight into a
// shared-memory plane, and k_node_pair's update of step n + 1 reads V from
// there instead of from HBM. Per node the step moves 80 B instead of 88 B
// and runs one kernel instead of two (V_{n+1} is never re-read, d_1 is read
// once, with its halo, from L2).
// March: iteration w produces W(w) (planes max(zb - 1, 0) .. min(ze, nz - 1);
// the chunk's own planes go to global memory) and then updates the nodes of
// plane z = w - 1 from W(z - 1), W(z), W(z + 1) (the thread's own column
// window) and the in-plane neighbours of W(z) published one iteration
// earlier (double-buffered plane, one __syncthreads per iteration).
// Arithmetic and order are k_vin_tma_r's (producer) and k_node_pair's
// (update): bitwise equal to the two-kernel step (tests/test_gpu_xstep.py).
// ---------------------------------------------------------------------------
constexpr int kXDX = kPairTX + 4, kXDY = kPairTY + 4;   // d_1 box 68 x 8 (x0 - 2, y0 - 2)
constexpr int kXDT = kXDX * kXDY;
constexpr int kXDS = (kXDT + 15) & ~15;
constexpr int kXRD = 8;                                  // d_1 ring planes
constexpr int kXLA = 3;                                  // groups in flight ahead
constexpr int kXWS = kPairVS;                            // W plane (68 x 6)
constexpr size_t xstep_smem_bytes() {
  return sizeof(double) * (kXRD * kXDS + 2 * kXWS + kRG * 3 * kPairCS) + 128;
}

// A pair of x-adjacent cells of the producer: indices in a d_1 plane (cell 0
// and its mirrored in-plane neighbours), offset of cell 0 in a global plane.
struct XPairIdx {
  int c, xm, xp, ym, yp;
  long long gi;
  bool on;  // inside the grid
};
__device__ __forceinline__ XPairIdx x_pair_idx(const Geom& g, int x0, int y0, int row, int pr) {
  // row 0..5 of the W plane (gy = y0 - 1 + row), pair 0..33 (gx = x0 - 2 + 2 pr)
  XPairIdx q;
  const int gx = x0 - 2 + 2 * pr, gy = y0 - 1 + row;
  q.on = gx >= 0 && gx < g.n0 && gy >= 0 && gy < g.n1;
  q.c = (row + 1) * kXDX + 2 * pr;
  q.xm = q.c + ((gx > 0 && pr > 0) ? -1 : 1);
  q.xp = q.c + 1 + ((gx + 1 < g.n0 - 1 && pr < 33) ? 1 : -1);
  q.ym = q.c + (gy > 0 ? -kXDX : kXDX);
  q.yp = q.c + (gy < g.n1 - 1 ? kXDX : -kXDX);
  q.gi = (long long)gx + (long long)g.n0 * gy;
  return q;
}

// W of a pair at plane w from the d_1 planes (lower, centre, upper of the
// pair's column; in-plane neighbours from the centre plane DC) and V_n.
__device__ __forceinline__ void x_produce(const Geom& g, const XArgs& a, const double* DC,
                                          const XPairIdx& q, double2 dm, double2 dc, double2 dp,
                                          double2 vn, double2& dk, double2& o) {
  const double2 ym = *reinterpret_cast<const double2*>(DC + q.ym);
  const double2 yp = *reinterpret_cast<const double2*>(DC + q.yp);
  const double xm0 = DC[q.xm], xp1 = DC[q.xp];
  double L0 = fma(g.wc, dc.x, g.w[2] * (dm.x + dp.x));
  double L1 = fma(g.wc, dc.y, g.w[2] * (dm.y + dp.y));
  L0 = fma(g.w[0], xm0 + dc.y, L0);
  L1 = fma(g.w[0], dc.x + xp1, L1);
  L0 = fma(g.w[1], ym.x + yp.x, L0);
  L1 = fma(g.w[1], ym.y + yp.y, L1);
  dk.x = fma(a.mueta2, fma(dc.x, a.inv_mue1, L0), a.nu2 * dc.x);
  dk.y = fma(a.mueta2, fma(dc.y, a.inv_mue1, L1), a.nu2 * dc.y);
  o.x = fma(a.cG2, dk.x, vn.x);
  o.y = fma(a.cG2, dk.y, vn.y);
}

// V_{n+1} at in-plane offset j of plane zz, from the complete fields d_1^n
// and V_n (rare paths: deferred planes, abort ordinal).
__device__ __noinline__ double x_w_at(const Geom& g, const XArgs& a, long long j, int zz) {
  const int nz = g.nzl;
  const double* Dn = a.d1;
  const int gx = (int)(j % g.n0), gy = (int)(j / g.n0);
  const long long xm = gx > 0 ? -1 : 1, xp = gx < g.n0 - 1 ? 1 : -1;
  const long long ym = gy > 0 ? -(long long)g.n0 : (long long)g.n0;
  const long long yp = gy < g.n1 - 1 ? (long long)g.n0 : -(long long)g.n0;
  const int zm = zz > 0 ? zz - 1 : 1, zp = zz < nz - 1 ? zz + 1 : nz - 2;
  const long long k0 = j + g.plane * zz;
  const double dcv = __ldg(Dn + k0);
  double L = fma(g.wc, dcv, g.w[2] * (__ldg(Dn + j + g.plane * zm) + __ldg(Dn + j + g.plane * zp)));
  L = fma(g.w[0], __ldg(Dn + k0 + xm) + __ldg(Dn + k0 + xp), L);
  L = fma(g.w[1], __ldg(Dn + k0 + ym) + __ldg(Dn + k0 + yp), L);
  const double dkv = fma(a.mueta2, fma(dcv, a.inv_mue1, L), a.nu2 * dcv);
  return fma(a.cG2, dkv, __ldg(a.vn + k0));
}
// Stencil inputs of the update at column offset j, plane z.
struct XStencil {
  double vm, vc, vp, xs, ys;
};
__device__ __forceinline__ XStencil x_stencil(const Geom& g, const XArgs& a, long long j, int z) {
  const int nz = g.nzl;
  const int gx = (int)(j % g.n0), gy = (int)(j / g.n0);
  const long long xm = gx > 0 ? -1 : 1, xp = gx < g.n0 - 1 ? 1 : -1;
  const long long ym = gy > 0 ? -(long long)g.n0 : (long long)g.n0;
  const long long yp = gy < g.n1 - 1 ? (long long)g.n0 : -(long long)g.n0;
  XStencil s;
  s.vc = x_w_at(g, a, j, z);
  s.vm = x_w_at(g, a, j, z > 0 ? z - 1 : 1);
  s.vp = x_w_at(g, a, j, z < nz - 1 ? z + 1 : nz - 2);
  s.xs = x_w_at(g, a, j + xm, z) + x_w_at(g, a, j + xp, z);
  s.ys = x_w_at(g, a, j + ym, z) + x_w_at(g, a, j + yp, z);
  return s;
}
// inner_nonfinite of a column (P/src/cheb.cpp:73-80, multirate.cpp:100-104)
// with V of y_{n+1} recomputed (other blocks may still be writing theirs).
__device__ __noinline__ bool x_inner_nonfinite(const Geom& g, const XArgs& a, long long j, int z0,
                                               int z1) {
  bool inner = false;
  const double* G = a.f.g1;
  for (int z = z0; z < z1; ++z) {
    const XStencil s = x_stencil(g, a, j, z);
    double D = fma(g.wc, s.vc, g.w[2] * (s.vm + s.vp));
    D = fma(g.w[0], s.xs, D);
    D = fma(g.w[1], s.ys, D);
    const long long i = j + g.plane * z;
    const double q0 = __ldg(G + g.nn + i), q1 = __ldg(G + 2 * g.nn + i), q2 = __ldg(G + 3 * g.nn + i);
    const Dgate d = hh_expeuler_ref(s.vc, q0, q1, q2, a.f.eta);
    const double y0 = q0 + d.d0, y1 = q1 + d.d1, y2 = q2 + d.d2;
    const double fs = -current_fast(s.vc, y0, y1, y2) * g.inv_Cm;
    inner |= !(finite_hi(D + fs) && finite_hi(y0) && finite_hi(y1) && finite_hi(y2));
  }
  return inner;
}

__global__ void __launch_bounds__(kPairNT, 3)
    k_step_x(const Geom g, const XArgs a, const __grid_constant__ TmaX tm) {
  constexpr int CS = kPairCS, HXT = kPairHX;
  const FastArgs& f = a.f;
  extern __shared__ __align__(128) double smem_tma[];
  double* dst = smem_tma + ((128u - (smem_u32(smem_tma) & 127u)) & 127u) / 8;  // [kXRD][kXDS]
  double* wst = dst + kXRD * kXDS;   // [2][kXWS]
  double* gst = wst + 2 * kXWS;      // [kRG][3][CS]
  __shared__ double tab[256];
  __shared__ __align__(8) unsigned long long bars[8];
  __shared__ int skip;
  const int t = threadIdx.x;
  const int nz = g.nzl;
  const int zb = blockIdx.z * f.zc;
  const int ze = min(nz, zb + f.zc);
  pdl_launch_dependents();
  if (t == 0) {
    for (int s = 0; s < 8; ++s) mbar_init(smem_u32(&bars[s]), 1);
    mbar_fence_init();
    prefetch_tensormap(&tm.d1);
    prefetch_tensormap(&tm.gates);
  }
  __syncthreads();
  const int px = t & 31, ty = t >> 5;
  const int x0 = blockIdx.x * kPairTX, y0 = blockIdx.y * kPairTY;
  const int cx = x0 + 2 * px, cy = y0 + ty;
  const bool valid = cx < g.n0 && cy < g.n1;
  const long long ip = valid ? (long long)cx + (long long)g.n0 * cy : 0;
  const long long nn = g.nn, plane = g.plane;
  const unsigned d0 = smem_u32(dst), gs0 = smem_u32(gst), b0 = smem_u32(bars);
  const int w0 = zb > 0 ? zb - 1 : 0;          // first W plane produced
  const int w1 = min(ze, nz - 1);              // last W plane produced
  const int pbase = w0 - 1;                    // d_1 ring: slot (p - pbase) & 7
  auto dslot = [&](int p) { return (p - pbase) & (kXRD - 1); };
  // group of iteration w: d_1 of plane w + 1 (the producer's upper plane) and
  // the gates of plane w - 1 (the update's plane)
  auto group_bytes = [&](int w) {
    unsigned b = 0;
    if (w <= w1 && w + 1 <= nz - 1) b += 8u * kXDT;
    if (w - 1 >= zb && w - 1 < ze) b += 8u * 3 * CS;
    return b;
  };
  auto issue_group = [&](int w, unsigned extra) {  // thread 0
    const unsigned bar = b0 + 8u * ((w - w0) & 7);
    mbar_expect_tx(bar, group_bytes(w) + extra);
    if (w <= w1 && w + 1 <= nz - 1)
      tma_load_3d(d0 + 8u * kXDS * dslot(w + 1), &tm.d1, bar, x0 - 2, y0 - 2, w + 1);
    if (w - 1 >= zb && w - 1 < ze)
      tma_load_4d(gs0 + 8u * 3 * CS * ((w - 1 - zb) & (kRG - 1)), &tm.gates, bar, x0, y0, w - 1, 1);
  };
  pdl_wait();
  if (t == 0) {
    // first group: also d_1 of planes w0 - 1 (if any) and w0, and the exp table
    unsigned extra = sizeof(double) * 256 + 8u * kXDT + (w0 >= 1 ? 8u * kXDT : 0u);
    issue_group(w0, extra);
    const unsigned bar = b0;
    bulk_load(smem_u32(tab), kExp2Tab256, sizeof(double) * 256, bar);
    tma_load_3d(d0 + 8u * kXDS * dslot(w0), &tm.d1, bar, x0 - 2, y0 - 2, w0);
    if (w0 >= 1) tma_load_3d(d0 + 8u * kXDS * dslot(w0 - 1), &tm.d1, bar, x0 - 2, y0 - 2, w0 - 1);
    for (int i = 1; i < kXLA && w0 + i <= ze; ++i) issue_group(w0 + i, 0);
  }
  if (t == 32) skip = (*(volatile const unsigned long long*)f.event) < a.code_prev + 2;
  __syncthreads();
  if (skip != 0) {  // an earlier step aborted: drain the prologue copies
    for (int i = 0; i < kXLA && w0 + i <= ze; ++i) mbar_wait(b0 + 8u * i, 0);
    return;
  }
  // producer pairs: the thread's own (interior) pair, row ty + 1, pair px + 1;
  // threads 0..75 also take one pair of the one-cell halo ring
  const XPairIdx qi = x_pair_idx(g, x0, y0, ty + 1, px + 1);
  XPairIdx qe;
  qe.on = false;
  if (t < 76) {
    const int row = t < 34 ? 0 : (t < 68 ? 5 : 1 + ((t - 68) >> 1));
    const int pr = t < 34 ? t : (t < 68 ? t - 34 : (((t - 68) & 1) ? 33 : 0));
    qe = x_pair_idx(g, x0, y0, row, pr);
  }
  // update: cell 0 of the pair in a W plane and its mirrored neighbours
  const int cell = (ty + 1) * HXT + 2 * px + 2;
  const int cxm = cell + (cx > 0 ? -1 : 1), cxp = cell + 1 + (cx + 1 < g.n0 - 1 ? 1 : -1);
  const int cym = cell + (cy > 0 ? -HXT : HXT), cyp = cell + (cy < g.n1 - 1 ? HXT : -HXT);
  const int gcell = ty * kPairTX + 2 * px;
  int zs0 = 1, zs1 = 0;
  const bool st0 = valid && stim_col_xy<3>(g, cx, cy), st1 = valid && stim_col_xy<3>(g, cx + 1, cy);
  if (st0 || st1) {
    zs0 = g.st_lo[2] - g.zoff;
    zs1 = g.st_hi[2] - g.zoff;
  }
  // step n (producer) events; step n + 1 (update) events and gate range
  bool p_bad_in = false, p_bad_out = false, p_guard = false;
  double glo = 2.0, ghi = -1.0;
  unsigned tlo = 0xffffffffu, thi = 0u;
  unsigned long long plo = ~0ull, phi = 0ull;
  if (f.last && f.gate_prev) {
    plo = f.gate_prev[0];
    phi = f.gate_prev[1];
    const unsigned hl = (unsigned)((plo ^ 0x8000000000000000ull) >> 32);
    const unsigned hh = (unsigned)((phi ^ 0x8000000000000000ull) >> 32);
    if (plo != ~0ull && (plo >> 63) && (phi >> 63) && hh < 0x7ff00000u && hl <= hh) {
      tlo = hl;
      thi = hh;
      glo = __longlong_as_double((long long)(plo ^ 0x8000000000000000ull));
      ghi = __longlong_as_double((long long)(phi ^ 0x8000000000000000ull));
    } else {
      plo = ~0ull;
      phi = 0ull;
    }
  }
  unsigned nfacc = 0u;
  unsigned long long slow_mask = 0;
  mbar_wait(b0, 0);  // d_1 of w0 - 1, w0, w0 + 1, gates of w0 - 1, table
  // d_1 window of the own pair: planes w - 1, w (w = w0)
  double2 dm = make_double2(0.0, 0.0), dc;
  if (w0 >= 1) dm = *reinterpret_cast<const double2*>(dst + dslot(w0 - 1) * kXDS + qi.c);
  dc = *reinterpret_cast<const double2*>(dst + dslot(w0) * kXDS + qi.c);
  double2 wm = make_double2(0.0, 0.0), wc = make_double2(0.0, 0.0);  // W(z - 1), W(z)
  double* po = f.out + ip + plane * zb;   // gates of y_{n+2}
  double* pu = f.u1 + ip + plane * zb;    // d_1 of step n + 1
  // V_n of the pairs two planes ahead (global loads: under load their latency
  // exceeds one iteration)
  const double2 zero2 = make_double2(0.0, 0.0);
  auto ld_vn = [&](int w) {
    return (valid && w <= w1) ? __ldg(reinterpret_cast<const double2*>(a.vn + ip + plane * w)) : zero2;
  };
  auto ld_ev = [&](int w) {
    return (qe.on && w >= zb && w < ze && w <= w1)
               ? __ldg(reinterpret_cast<const double2*>(a.vn + qe.gi + plane * w))
               : zero2;
  };
  double2 vn = ld_vn(w0), ev = ld_ev(w0);
  double2 vn1 = ld_vn(w0 + 1), ev1 = ld_ev(w0 + 1);
  for (int w = w0; w <= ze; ++w) {
    const int it = w - w0;
    if (t == 0 && w + kXLA <= ze) issue_group(w + kXLA, 0);
    const double2 vn2 = ld_vn(w + 2), ev2 = ld_ev(w + 2);
    if (it > 0) mbar_wait(b0 + 8u * (it & 7), (it >> 3) & 1);
    // ---- producer: W(w) ----
    double2 wp = make_double2(0.0, 0.0);
    if (w <= w1) {
      const double* DC = dst + dslot(w) * kXDS;
      double2 dp;
      if (w + 1 <= nz - 1) dp = *reinterpret_cast<const double2*>(dst + dslot(w + 1) * kXDS + qi.c);
      else dp = dm;              // mirror at the top face
      if (w == 0) dm = dp;       // mirror at the bottom face
      const bool ownp = w >= zb && w < ze;
      double2 dk;
      x_produce(g, a, DC, qi, dm, dc, dp, vn, dk, wp);
      *reinterpret_cast<double2*>(wst + (w & 1) * kXWS + qi.c - kXDX) = wp;
      if (ownp && valid) {
        *reinterpret_cast<double2*>(a.vout + ip + plane * w) = wp;
        p_bad_in |= !finite_hi(dk.x) || !finite_hi(dk.y);
        p_bad_out |= !finite_hi(wp.x) || !finite_hi(wp.y);
        p_guard |= !(fabs(wp.x) <= 1e6) || !(fabs(wp.y) <= 1e6);
      }
      dm = dc;
      dc = dp;
      if (ownp && qe.on) {  // the halo ring of the chunk's own planes
        const double* DM = dst + dslot(w == 0 ? 1 : w - 1) * kXDS;
        const double* DP = dst + dslot(w + 1 <= nz - 1 ? w + 1 : w - 1) * kXDS;
        const double2 em = *reinterpret_cast<const double2*>(DM + qe.c);
        const double2 ec = *reinterpret_cast<const double2*>(DC + qe.c);
        const double2 ep = *reinterpret_cast<const double2*>(DP + qe.c);
        double2 ek, eo;
        x_produce(g, a, DC, qe, em, ec, ep, ev, ek, eo);
        *reinterpret_cast<double2*>(wst + (w & 1) * kXWS + qe.c - kXDX) = eo;
      }
    }
    // ---- update of step n + 1: plane z = w - 1 ----
    const int z = w - 1;
    if (z >= zb) {
      double2 um = wm, up = wp;
      if (z == 0) um = wp;         // mirror at the bottom face
      if (z == nz - 1) up = wm;    // mirror at the top face
      const double* V0 = wst + (z & 1) * kXWS;
      const double2 ym = *reinterpret_cast<const double2*>(V0 + cym);
      const double2 yp = *reinterpret_cast<const double2*>(V0 + cyp);
      const double xm0 = V0[cxm], xp1 = V0[cxp];
      const double* G0 = gst + ((z - zb) & (kRG - 1)) * 3 * CS + gcell;
      const double2 za = *reinterpret_cast<const double2*>(G0);
      const double2 zb2 = *reinterpret_cast<const double2*>(G0 + CS);
      const double2 zc2 = *reinterpret_cast<const double2*>(G0 + 2 * CS);
      const int hx = __double2hiint(wc.x), hy = __double2hiint(wc.y);
      const bool fast = hx < f.vq_pos && (unsigned)hx < f.vq_neg && hy < f.vq_pos &&
                        (unsigned)hy < f.vq_neg;
      if (!fast) slow_mask |= 1ull << (z - zb);
      NodeOut r0 = node_update_s<3, 1, 1, 0>(g, f, tab, um.x, wc.x, up.x, xm0 + wc.y, ym.x + yp.x,
                                             za.x, zb2.x, zc2.x, 0.0, nullptr, 0);
      NodeOut r1 = node_update_s<3, 1, 1, 0>(g, f, tab, um.y, wc.y, up.y, wc.x + xp1, ym.y + yp.y,
                                             za.y, zb2.y, zc2.y, 0.0, nullptr, 0);
      if (z >= zs0 && z <= zs1) {
        if (st0) r0.o0 = fma(f.mue1, f.stim, r0.o0);
        if (st1) r1.o0 = fma(f.mue1, f.stim, r1.o0);
      }
      if (valid && fast) {
        *reinterpret_cast<double2*>(po + nn) = make_double2(r0.o1, r1.o1);
        *reinterpret_cast<double2*>(po + 2 * nn) = make_double2(r0.o2, r1.o2);
        *reinterpret_cast<double2*>(po + 3 * nn) = make_double2(r0.o3, r1.o3);
        *reinterpret_cast<double2*>(pu) = make_double2(r0.o0, r1.o0);
        nfacc = max(max(nfacc, max(nf_hi(r0.o0), nf_hi(r0.o1))), max(nf_hi(r0.o2), nf_hi(r0.o3)));
        nfacc = max(max(nfacc, max(nf_hi(r1.o0), nf_hi(r1.o1))), max(nf_hi(r1.o2), nf_hi(r1.o3)));
        bool track = f.last;
        if (track) {
          const unsigned h0 = __double2hiint(r0.o1), h1 = __double2hiint(r0.o2),
                         h2 = __double2hiint(r0.o3), h3 = __double2hiint(r1.o1),
                         h4 = __double2hiint(r1.o2), h5 = __double2hiint(r1.o3);
          const unsigned hmin = min(min(min(h0, h1), min(h2, h3)), min(h4, h5));
          const unsigned hmax = max(max(max(h0, h1), max(h2, h3)), max(h4, h5));
          track = hmin <= tlo || hmax >= thi;
        }
        if (track) {
          glo = r0.o1 < glo ? r0.o1 : glo;
          ghi = ghi < r0.o1 ? r0.o1 : ghi;
          glo = r0.o2 < glo ? r0.o2 : glo;
          ghi = ghi < r0.o2 ? r0.o2 : ghi;
          glo = r0.o3 < glo ? r0.o3 : glo;
          ghi = ghi < r0.o3 ? r0.o3 : ghi;
          glo = r1.o1 < glo ? r1.o1 : glo;
          ghi = ghi < r1.o1 ? r1.o1 : ghi;
          glo = r1.o2 < glo ? r1.o2 : glo;
          ghi = ghi < r1.o2 ? r1.o2 : ghi;
          glo = r1.o3 < glo ? r1.o3 : glo;
          ghi = ghi < r1.o3 ? r1.o3 : ghi;
        }
      }
      po += plane;
      pu += plane;
    }
    wm = wc;
    wc = wp;
    vn = vn1;
    ev = ev1;
    vn1 = vn2;
    ev1 = ev2;
    __syncthreads();
  }
  // ---- events of step n (inner stage 2, outer stage, norm guard) ----
  if (p_bad_in) atomicMin(f.event, a.code_prev + 2ull);
  if (p_bad_out) atomicMin(f.event, a.code_prev + 3ull);
  if (p_guard) atomicMin(f.event, a.code_prev + 4ull);
  // ---- step n + 1: deferred planes, events, gate range (as k_node_pair) ----
  bool bad = nfacc == 0xffffffffu;
  if (valid && slow_mask) {  // planes deferred by the window test: per-node path
    for (int c = 0; c < 2; ++c) {
      const long long ipc = ip + c;
      const double* G = f.g1;
      const bool stc = c ? st1 : st0;
      for (int z = zb; z < ze; ++z) {
        if (!(slow_mask >> (z - zb) & 1ull)) continue;
        const long long i = ipc + plane * z;
        const XStencil sx = x_stencil(g, a, ipc, z);
        const double stim = (stc && z >= zs0 && z <= zs1) ? f.stim : 0.0;
        double q[4] = {0.0, 0.0, 0.0, 0.0};
        NodeOut r;
        if (fabs(sx.vc - f.vmid) <= f.vfast) {  // the hot loop's form (stimulus added after)
          r = node_update_s<3, 1, 1, 0>(g, f, tab, sx.vm, sx.vc, sx.vp, sx.xs, sx.ys,
                                        __ldg(G + nn + i), __ldg(G + 2 * nn + i),
                                        __ldg(G + 3 * nn + i), 0.0, q, 1);
          if (stc && z >= zs0 && z <= zs1) r.o0 = fma(f.mue1, f.stim, r.o0);
        } else {
          r = node_update_s<3, 1, 1, 1>(g, f, tab, sx.vm, sx.vc, sx.vp, sx.xs, sx.ys,
                                        __ldg(G + nn + i), __ldg(G + 2 * nn + i),
                                        __ldg(G + 3 * nn + i), stim, q, 1);
        }
        f.out[nn + i] = r.o1;
        f.out[2 * nn + i] = r.o2;
        f.out[3 * nn + i] = r.o3;
        f.u1[i] = r.o0;
        bad |= !finite_hi((r.o0 + r.o1) + (r.o2 + r.o3));
        if (f.last) {
          glo = fmin(glo, fmin(r.o1, fmin(r.o2, r.o3)));
          ghi = fmax(ghi, fmax(r.o1, fmax(r.o2, r.o3)));
        }
      }
    }
  }
  if (bad && !f.exex) {  // exact ordinal: inner stage 1 before the outer stage
    const bool inner = x_inner_nonfinite(g, a, ip, zb, ze) || x_inner_nonfinite(g, a, ip + 1, zb, ze);
    atomicMin(f.event, f.code_base + (inner ? 1ull : (unsigned long long)(f.m + 1)));
  }
  if (f.last) {
    unsigned long long lo = valid && ze > zb ? ord_of(glo) : ~0ull;
    unsigned long long hi = valid && ze > zb ? ord_of(ghi) : 0ull;
    block_gate_range(f.gate_slot, min(lo, plo), max(hi, phi));
  }
}

// ---------------------------------------------------------------------------
// k_resident: a whole emrkc_run on a small grid in one cooperative launch
// (s = m = 1). Config 1 (256^2) and the small sweep grids are launch- and
// latency-bound one step per launch (~11 us for 65k nodes); here every
// thread owns R nodes for the whole run (gates in registers, old and new for
// the abort rollback), V ping-pongs through vbuf (L2-resident, read with
// ld.global.cg so no stale L1 line survives a step), and one grid barrier
// per step (a monotonic arrival counter; cooperative launch guarantees
// co-residency) publishes V and the step's abort ordinal. The run-loop
// semantics are the per-step kernels' (P/src/simulate.cpp:176-229): a
// non-finite step leaves the pre-step state, a norm-guard step keeps its
// result, later steps do not run; the gate range over the accepted steps
// goes to slot 0, which the host folds like the per-step slots.
// ---------------------------------------------------------------------------
constexpr int kResNT = 256;
template <int DIM, int R>
__global__ void __launch_bounds__(kResNT) k_resident(const Geom g, const ResidentArgs ra) {
  const FastArgs& a = ra.f;
  __shared__ double tab[256];
  __shared__ unsigned long long ev_sh;
  __shared__ unsigned long long rlo[kResNT / 32], rhi[kResNT / 32];
  const int t = threadIdx.x;
  load_exp_table(tab, t, kResNT);
  const long long nn = g.nn;
  const long long b0 = nn * blockIdx.x / gridDim.x, b1 = nn * (blockIdx.x + 1) / gridDim.x;
  // node k of this thread: b0 + t + k * NT; flags: bit0 x>0, bit1 x<n0-1,
  // bit2 y>0, bit3 y<n1-1, bit4 z>0, bit5 z<n2-1, bit6 in the stimulus box
  long long idx[R];
  unsigned fl[R];
  double z0[R], z1[R], z2[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    idx[k] = b0 + t + (long long)k * kResNT;
    fl[k] = 0;
    z0[k] = z1[k] = z2[k] = 0.0;
    if (idx[k] < b1) {
      const long long i = idx[k];
      const int x = (int)(i % g.n0);
      const int y = DIM == 3 ? (int)((i / g.n0) % g.n1) : (int)(i / g.n0);
      const int zz = DIM == 3 ? (int)(i / g.plane) : 0;
      fl[k] = (x > 0 ? 1u : 0u) | (x < g.n0 - 1 ? 2u : 0u) | (y > 0 ? 4u : 0u) |
              (y < (DIM == 3 ? g.n1 : g.nzg) - 1 ? 8u : 0u);
      if (DIM == 3) fl[k] |= (zz > 0 ? 16u : 0u) | (zz < g.nzg - 1 ? 32u : 0u);
      const bool box = DIM == 3 ? (stim_col_xy<3>(g, x, y) && zz >= g.st_lo[2] && zz <= g.st_hi[2])
                                : (stim_col_xy<2>(g, x, y) && y >= g.st_lo[1] && y <= g.st_hi[1]);
      if (box) fl[k] |= 64u;
      z0[k] = ra.y_in[nn + i];
      z1[k] = ra.y_in[2 * nn + i];
      z2[k] = ra.y_in[3 * nn + i];
      ra.vbuf[i] = ra.y_in[i];
    }
  }
  // vbuf[0] complete before any block reads a neighbour (arrival 0)
  __syncthreads();
  if (t == 0) {
    __threadfence();
    atomicAdd(ra.bar + 1, 1u);
    while (ld_acquire_gpu_u32(ra.bar + 1) < gridDim.x) {
    }
  }
  __syncthreads();
  const long long sx = 1, sy = g.n0, sz = DIM == 3 ? g.plane : 0;
  // the slab axis (z in 3-D, y in 2-D) is the stencil's "vm/vp" direction
  const long long sv = DIM == 3 ? sz : sy;
  long long r = 0;
  int fin = 0;      // buffer holding the final V
  double rglo = 2.0, rghi = -1.0;  // gate range over the accepted steps
  bool rany = false;
  bool keep_new = false;
  double n0v[R], n1v[R], n2v[R];
  for (; r < ra.nsteps; ++r) {
    const double* V = ra.vbuf + (r & 1) * nn;
    double* Vn = ra.vbuf + ((r + 1) & 1) * nn;
    const double stim = ra.stim[r];
    const unsigned long long cb = (unsigned long long)r * ra.stride;
    bool inner_bad = false, outer_bad = false, guard = false;
    double glo = 2.0, ghi = -1.0;
    bool any = false;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      n0v[k] = z0[k];
      n1v[k] = z1[k];
      n2v[k] = z2[k];
      if (idx[k] >= b1) continue;
      const long long i = idx[k];
      const unsigned f = fl[k];
      const double vc = __ldcg(V + i);
      // slab-axis neighbours (mirror at the boundary, P/src/monodomain.cpp:85-86)
      const unsigned bm = DIM == 3 ? 16u : 4u, bp = DIM == 3 ? 32u : 8u;
      const double vm = __ldcg(V + i + ((f & bm) ? -sv : sv));
      const double vp = __ldcg(V + i + ((f & bp) ? sv : -sv));
      const double xs = __ldcg(V + i + ((f & 1u) ? -sx : sx)) + __ldcg(V + i + ((f & 2u) ? sx : -sx));
      double ys = 0.0;
      if (DIM == 3) ys = __ldcg(V + i + ((f & 4u) ? -sy : sy)) + __ldcg(V + i + ((f & 8u) ? sy : -sy));
      const bool box = (f & 64u) != 0;
      const bool fast = fabs(vc - a.vmid) <= a.vfast;
      NodeOut o;
      if (fast) {
        o = node_update_s<DIM, 1, 0, 0>(g, a, tab, vm, vc, vp, xs, ys, z0[k], z1[k], z2[k], 0.0,
                                         nullptr, 1);
        if (box) o.o0 = fma(a.cV, stim, o.o0);
      } else {  // k_node_tma's deferred-node arithmetic
        double q[4] = {0.0, 0.0, 0.0, 0.0};
        o = node_update_s<DIM, 1, 0, 1>(g, a, tab, vm, vc, vp, xs, ys, z0[k], z1[k], z2[k],
                                         box ? stim : 0.0, q, 1);
      }
      Vn[i] = o.o0;
      n0v[k] = o.o1;
      n1v[k] = o.o2;
      n2v[k] = o.o3;
      guard |= !(fabs(o.o0) <= 1e6);
      if (!finite_hi((o.o0 + o.o1) + (o.o2 + o.o3)) && !a.exex) {
        // inner stage 1 is checked before the outer stage (P/src/cheb.cpp:73-80)
        double D = fma(g.wc, vc, g.w[DIM - 1] * (vp + vm));
        if (DIM >= 2) D = fma(g.w[0], xs, D);
        if (DIM == 3) D = fma(g.w[1], ys, D);
        const Dgate d = hh_expeuler_ref(vc, z0[k], z1[k], z2[k], a.eta);
        const double y0 = z0[k] + d.d0, y1 = z1[k] + d.d1, y2 = z2[k] + d.d2;
        const double fs = -current_fast(vc, y0, y1, y2) * g.inv_Cm;
        if (!(finite_hi(D + fs) && finite_hi(y0) && finite_hi(y1) && finite_hi(y2)))
          inner_bad = true;
        else
          outer_bad = true;
      }
      any = true;
      glo = o.o1 < glo ? o.o1 : glo;
      ghi = ghi < o.o1 ? o.o1 : ghi;
      glo = o.o2 < glo ? o.o2 : glo;
      ghi = ghi < o.o2 ? o.o2 : ghi;
      glo = o.o3 < glo ? o.o3 : glo;
      ghi = ghi < o.o3 ? o.o3 : ghi;
    }
    if (inner_bad) atomicMin(a.event, cb + 1ull);
    else if (outer_bad) atomicMin(a.event, cb + 2ull);
    if (guard) atomicMin(a.event, cb + 3ull);
    // grid barrier: a monotonic arrival counter (zeroed by the host); the
    // abort word is read by the arriving thread once everyone is in, so
    // the step's V and its abort ordinal are published together
    __syncthreads();  // the block's V stores and abort atomics are done
    if (t == 0) {
      __threadfence();
      atomicAdd(ra.bar, 1u);
      const unsigned target = (unsigned)(r + 1) * gridDim.x;
      while (ld_acquire_gpu_u32(ra.bar) < target) {
      }
      ev_sh = *(volatile const unsigned long long*)a.event;
    }
    __syncthreads();
    const unsigned long long ev = ev_sh;
    if (ev != kNoEvent) {  // this step raised an event (earlier ones did not)
      if (ev - cb == 3ull) {  // norm guard: the step's result is the state
        fin = (int)((r + 1) & 1);
        keep_new = true;
      } else {                // NumericalAbort: the pre-step state
        fin = (int)(r & 1);
      }
      break;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      z0[k] = n0v[k];
      z1[k] = n1v[k];
      z2[k] = n2v[k];
    }
    if (any) {  // an accepted step: into the run's gate range (simulate.cpp:228)
      rglo = glo < rglo ? glo : rglo;
      rghi = rghi < ghi ? ghi : rghi;
      rany = true;
    }
  }
  {  // the run's gate range over its accepted steps -> slot 0 (the host folds
     // slots 0 .. accepted - 1; the others stay empty)
    unsigned long long lo = rany ? ord_of(rglo) : ~0ull, hi = rany ? ord_of(rghi) : 0ull;
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((t & 31) == 0) {
      rlo[t >> 5] = lo;
      rhi[t >> 5] = hi;
    }
    __syncthreads();
    if (t == 0) {
      for (int w = 1; w < kResNT / 32; ++w) {
        lo = min(lo, rlo[w]);
        hi = max(hi, rhi[w]);
      }
      if (lo != ~0ull) atomicMin(ra.slots, lo);
      if (hi != 0ull) atomicMax(ra.slots + 1, hi);
    }
  }
  if (r == ra.nsteps) fin = (int)(r & 1);
  const double* Vf = ra.vbuf + fin * nn;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (idx[k] >= b1) continue;
    const long long i = idx[k];
    ra.y_out[i] = __ldcg(Vf + i);
    ra.y_out[nn + i] = keep_new ? n0v[k] : z0[k];
    ra.y_out[2 * nn + i] = keep_new ? n1v[k] : z1[k];
    ra.y_out[3 * nn + i] = keep_new ? n2v[k] : z2[k];
  }
}

template <int DIM, int R>
static int resident_blocks() {
  static int nb = -1;
  if (nb < 0) {
    int per = 0, dev = 0, nsm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_resident<DIM, R>, kResNT, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    nb = per * nsm;
  }
  return nb;
}

template <int DIM, int R>
static cudaError_t launch_resident_t(const Geom& g, const ResidentArgs& a, cudaStream_t st) {
  const int nb = resident_blocks<DIM, R>();
  // fewest blocks that keep R nodes per thread, at most one wave
  long long want = (g.nn + (long long)kResNT * R - 1) / ((long long)kResNT * R);
  if (want > nb) return cudaErrorInvalidValue;
  // spread over every SM when the grid allows (shorter per-step chains)
  if (want < nb) want = std::min<long long>(nb, (g.nn + kResNT - 1) / kResNT);
  Geom gg = g;
  ResidentArgs aa = a;
  void* args[] = {&gg, &aa};
  return cudaLaunchCooperativeKernel((const void*)k_resident<DIM, R>, dim3((unsigned)want),
                                     dim3(kResNT), args, 0, st);
}

}  // namespace

long long resident_capacity(int dim) {
  if (dim == 3) return (long long)resident_blocks<3, 4>() * kResNT * 4;
  if (dim == 2) return (long long)resident_blocks<2, 4>() * kResNT * 4;
  return 0;
}

cudaError_t launch_resident(const Geom& g, const ResidentArgs& a, cudaStream_t st) {
  // R nodes per thread: the smallest that fits one co-resident wave
  if (g.dim == 3) {
    if (g.nn <= (long long)resident_blocks<3, 1>() * kResNT) return launch_resident_t<3, 1>(g, a, st);
    if (g.nn <= (long long)resident_blocks<3, 2>() * kResNT * 2) return launch_resident_t<3, 2>(g, a, st);
    return launch_resident_t<3, 4>(g, a, st);
  }
  if (g.dim == 2) {
    if (g.nn <= (long long)resident_blocks<2, 1>() * kResNT) return launch_resident_t<2, 1>(g, a, st);
    if (g.nn <= (long long)resident_blocks<2, 2>() * kResNT * 2) return launch_resident_t<2, 2>(g, a, st);
    return launch_resident_t<2, 4>(g, a, st);
  }
  return cudaErrorInvalidValue;
}

namespace {

template <int DIM>
constexpr size_t tma_vin_smem_bytes() {
  using T = PipeTile<DIM>;
  return sizeof(double) * (kRV * TmaTile<DIM>::VS + kRG * 4 * T::NT) + 128;
}

template <int DIM, int LAST, int FIRST>
__global__ void __launch_bounds__(PipeTile<DIM>::NT, 7)
    k_vin_tma(const Geom g, const Halo h, const FastInnerArgs a, const __grid_constant__ TmaVin tm) {
  using T = PipeTile<DIM>;
  constexpr int VS = TmaTile<DIM>::VS;
  extern __shared__ __align__(128) double smem_tma[];
  // 128-byte aligned stage base (pointer arithmetic keeps the shared space)
  double* vst = smem_tma + ((128u - (smem_u32(smem_tma) & 127u)) & 127u) / 8;  // [kRV][VS]
  double* cst = vst + kRV * VS;                      // [kRG][4][NT]: d1, d_{k-2}, V1, V2
  __shared__ __align__(8) unsigned long long bars[kRV];
  __shared__ int skip;
  const int t = threadIdx.x;
  const int zb = a.z_lo + (DIM == 3 ? blockIdx.z : blockIdx.y) * a.zc;
  const int ze = min(a.z_hi, zb + a.zc);
  pdl_launch_dependents();
  if (t == 0) {
    for (int s = 0; s < kRV; ++s) mbar_init(smem_u32(&bars[s]), 1);
    mbar_fence_init();
    prefetch_tensormap(&tm.u);
  }
  __syncthreads();  // barriers initialised before any warp issues onto them
  const int tx = t % T::TX, ty = t / T::TX;
  const int x0 = blockIdx.x * T::TX;
  const int y0 = DIM == 3 ? blockIdx.y * T::TY : 0;
  const int cx = x0 + tx, cy = y0 + ty;
  const bool valid = cx < g.n0 && (DIM == 2 || cy < g.n1);
  const long long ip = valid ? (long long)cx + (long long)g.n0 * cy : 0;
  const long long plane = g.plane;
  const bool has2 = a.um2 != nullptr;
  const bool d1_is_u = a.um1 == a.d1;
  const unsigned v0 = smem_u32(vst), c0 = smem_u32(cst), b0 = smem_u32(bars);
  constexpr unsigned vbytes = 8u * TmaTile<DIM>::VT;
  const unsigned nb = (d1_is_u ? 0 : 1) + (has2 ? 1 : 0) + (LAST ? (FIRST ? 1 : 2) : 0);
  const unsigned cbytes = 8u * T::NT * nb;
  auto center = [&](const CUtensorMap* m, unsigned dst, unsigned bar, int zz) {
    if (DIM == 3) tma_load_3d(dst, m, bar, x0, y0, zz);
    else tma_load_2d(dst, m, bar, x0, zz);
  };
  // lane 0 of warp 0 (expect_tx + halo box), 1 (d_1, d_{k-2}), 2 (V of
  // g_{j-1}, g_{j-2}) issue a plane's copies
  const int role = (t & 31) == 0 ? (t >> 5) : -1;
  auto issue_comp = [&](int zz) {  // zz in [zb, ze)
    const int q = zz - zb + 1;
    const unsigned bar = b0 + 8u * (q & (kRV - 1));
    const unsigned sc = c0 + 8u * 4 * T::NT * ((zz - zb) & (kRG - 1));
    if (role == 0) {
      mbar_expect_tx(bar, vbytes + cbytes);
      const unsigned vd = v0 + 8u * VS * (q & (kRV - 1));
      if (DIM == 3) tma_load_3d(vd, &tm.u, bar, x0 - 2, y0 - 1, zz);
      else tma_load_2d(vd, &tm.u, bar, x0 - 2, zz);
    }
    if (role == (EMRKC_ISSUE1 ? 0 : 1)) {
      if (!d1_is_u) center(&tm.d1, sc, bar, zz);
      if (has2) center(&tm.um2, sc + 8u * T::NT, bar, zz);
    }
    if (LAST && role == (EMRKC_ISSUE1 ? 0 : 2)) {
      center(&tm.g1v, sc + 16u * T::NT, bar, zz);
      if (!FIRST) center(&tm.g2v, sc + 24u * T::NT, bar, zz);
    }
  };
  auto issue_edge = [&](int zz) {  // zz = zb - 1 or ze
    if (role != 0) return;
    const int q = zz - zb + 1;
    const unsigned bar = b0 + 8u * (q & (kRV - 1));
    mbar_expect_tx(bar, vbytes);
    tma_vplane<DIM>(g, &tm.u, &tm.glo, &tm.ghi, true, true, v0 + 8u * VS * (q & (kRV - 1)), bar,
                    x0, y0, zz);
  };
  pdl_wait();
  halo_wait(h, zb == 0, ze >= g.nzl);
  if (EMRKC_ISSUE1 ? role == 0 : (role >= 0 && role <= 2)) {
    // ghost planes arrived through generic peer stores (acquired in
    // halo_wait); order them before this thread's async-proxy reads
    if (role == 0) fence_proxy_async();
    issue_edge(zb - 1);
    for (int i = 0; i < kTmaLA; ++i) {
      if (zb + i < ze) issue_comp(zb + i);
      else {
        issue_edge(ze);
        break;
      }
    }
  }
  if (t == (EMRKC_EVWARP1 ? 32 : 0)) skip = (*(volatile const unsigned long long*)a.event) < level_floor(a.code_base, a.j, a.m, a.k);
  __syncthreads();
  const bool skipped = skip != 0;
  if (skipped) {  // aborted earlier: drain the prologue copies, release the neighbours
    const int np = 1 + min(kTmaLA, ze - zb) + (ze - zb < kTmaLA ? 1 : 0);
    for (int q = 0; q < np; ++q) mbar_wait(b0 + 8u * q, 0);
    halo_signal(h, zb == 0, ze >= g.nzl);
    return;
  }
  constexpr int HXT = TmaTile<DIM>::HX;
  const int cell = (DIM == 3 ? (ty + 1) * HXT : 0) + tx + 2;
  const int cxm = cell + (cx > 0 ? -1 : 1), cxp = cell + (cx < g.n0 - 1 ? 1 : -1);
  const int cym = cell + (cy > 0 ? -HXT : HXT), cyp = cell + (cy < g.n1 - 1 ? HXT : -HXT);
  bool bad_in = false, bad_out = false, guard = false;
  if (!skipped) {
    mbar_wait(b0, 0);
    mbar_wait(b0 + 8u, 0);
  }
  for (int z = zb; z < ze && !skipped; ++z) {
    const int p = z - zb + 1;
    if (EMRKC_ISSUE1 ? role == 0 : role >= 0) {
      if (z + kTmaLA < ze) issue_comp(z + kTmaLA);
      else if (z + kTmaLA == ze) issue_edge(ze);
    }
    mbar_wait(b0 + 8u * ((p + 1) & (kRV - 1)), ((p + 1) >> 3) & 1);
    const double* V0 = vst + (p & (kRV - 1)) * VS;
    const double vc = V0[cell];
    double D = fma(g.wc, vc, g.w[DIM - 1] * (vst[((p - 1) & (kRV - 1)) * VS + cell] +
                                             vst[((p + 1) & (kRV - 1)) * VS + cell]));
    if (DIM >= 2) D = fma(g.w[0], V0[cxm] + V0[cxp], D);
    if (DIM == 3) D = fma(g.w[1], V0[cym] + V0[cyp], D);
    const double* C0 = cst + ((z - zb) & (kRG - 1)) * 4 * T::NT + t;
    const double base = has2 ? fma(a.nu, vc, a.kappa * C0[T::NT]) : a.nu * vc;
    const double d1 = d1_is_u ? vc : C0[0];
    const double dk = fma(a.mueta, fma(d1, a.inv_mue1, D), base);
    if (valid) {
      const long long i = ip + plane * z;
      bad_in |= !finite_hi(dk);
      double vput = dk;
      if (!LAST) {
        a.uk[i] = dk;
      } else {
        const double gv = C0[2 * T::NT];
        const double bb = FIRST ? gv : fma(a.onu, gv, a.okappa * C0[3 * T::NT]);
        const double o0 = fma(a.cG, dk, bb);
        a.outv[i] = o0;
        bad_out |= !finite_hi(o0);
        guard |= !(fabs(o0) <= 1e6);  // also a non-finite V
        vput = o0;
      }
      if (z == 0 && h.put_lo) h.put_lo[ip] = vput;
      if (z == g.nzl - 1 && h.put_hi) h.put_hi[ip] = vput;
    }
    __syncthreads();
  }
  halo_signal(h, zb == 0, ze >= g.nzl);
  if (skipped) return;
  const unsigned long long base = a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1));
  if (bad_in) atomicMin(a.event, base + a.k);
  if (LAST && bad_out) atomicMin(a.event, base + a.m + 1);
  if (LAST && a.last && guard)
    atomicMin(a.event, a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
}

// ---------------------------------------------------------------------------
// k_vin_tma_r<LAST, FIRST, R>: k_vin_tma (3-D) with R rows per thread. The
// inner stages k >= 2 move 16-40 B per node and do ~12 FP64 operations, so
// one node per thread per plane left them issue-bound (75-85% issue, ncu):
// the per-plane work — mbarrier wait, ring-slot arithmetic, the plane
// barrier, thread 0's copy issue — cost more than the node. A 32 x 4R tile
// with 128 threads spreads that work over R nodes. The centre ring holds only
// the fields this launch reads (nb of d_1, d_{k-2}, V of g_{j-1}, g_{j-2}).
// Same arithmetic, in the same order, as k_vin_tma (bitwise equal).
// ---------------------------------------------------------------------------
#ifndef EMRKC_VIN_R
#define EMRKC_VIN_R 2
#endif
template <int R>
struct VinTileR {
  static constexpr int TX = 32, TY = 4 * R, NT = 128;
  static constexpr int CS = TX * TY;                 // centre cells
  static constexpr int HX = TX + 4, HY = TY + 2;
  static constexpr int VT = HX * HY;
  static constexpr int VS = (VT + 15) & ~15;
};
template <int R>
size_t tma_vin_r_smem_bytes(int nb) {
  return sizeof(double) * ((size_t)kRV * VinTileR<R>::VS + (size_t)kRG * nb * VinTileR<R>::CS) + 128;
}

template <int LAST, int FIRST, int R>
__global__ void __launch_bounds__(128)
    k_vin_tma_r(const Geom g, const Halo h, const FastInnerArgs a, const __grid_constant__ TmaVin tm) {
  using T = VinTileR<R>;
  constexpr int VS = T::VS;
  extern __shared__ __align__(128) double smem_tma[];
  double* vst = smem_tma + ((128u - (smem_u32(smem_tma) & 127u)) & 127u) / 8;  // [kRV][VS]
  double* cst = vst + kRV * VS;                      // [kRG][nb][CS]
  __shared__ __align__(8) unsigned long long bars[kRV];
  __shared__ int skip;
  const int t = threadIdx.x;
  const int zb = a.z_lo + blockIdx.z * a.zc;
  const int ze = min(a.z_hi, zb + a.zc);
  pdl_launch_dependents();
  if (t == 0) {
    for (int s = 0; s < kRV; ++s) mbar_init(smem_u32(&bars[s]), 1);
    mbar_fence_init();
    prefetch_tensormap(&tm.u);
  }
  __syncthreads();  // barriers initialised before any warp issues onto them
  const int tx = t % T::TX, ty = t / T::TX;  // rows ty, ty + 4, ...
  const int x0 = blockIdx.x * T::TX, y0 = blockIdx.y * T::TY;
  const long long plane = g.plane;
  const bool has2 = a.um2 != nullptr;
  const bool d1_is_u = a.um1 == a.d1;
  // centre fields present, packed: d_1, d_{k-2}, V of g_{j-1}, V of g_{j-2}
  const int f_um2 = d1_is_u ? 0 : 1;
  const int f_g1 = f_um2 + (has2 ? 1 : 0);
  const int nb = f_g1 + (LAST ? (FIRST ? 1 : 2) : 0);
  const unsigned v0 = smem_u32(vst), c0 = smem_u32(cst), b0 = smem_u32(bars);
  constexpr unsigned vbytes = 8u * T::VT;
  const unsigned cbytes = 8u * T::CS * nb;
  auto issue_comp = [&](int zz) {  // zz in [zb, ze); thread 0
    const int q = zz - zb + 1;
    const unsigned bar = b0 + 8u * (q & (kRV - 1));
    const unsigned sc = c0 + 8u * T::CS * nb * ((zz - zb) & (kRG - 1));
    mbar_expect_tx(bar, vbytes + cbytes);
    tma_load_3d(v0 + 8u * VS * (q & (kRV - 1)), &tm.u, bar, x0 - 2, y0 - 1, zz);
    if (!d1_is_u) tma_load_3d(sc, &tm.d1, bar, x0, y0, zz);
    if (has2) tma_load_3d(sc + 8u * T::CS * f_um2, &tm.um2, bar, x0, y0, zz);
    if (LAST) {
      tma_load_3d(sc + 8u * T::CS * f_g1, &tm.g1v, bar, x0, y0, zz);
      if (!FIRST) tma_load_3d(sc + 8u * T::CS * (f_g1 + 1), &tm.g2v, bar, x0, y0, zz);
    }
  };
  auto issue_edge = [&](int zz) {  // zz = zb - 1 or ze; thread 0
    const int q = zz - zb + 1;
    const unsigned bar = b0 + 8u * (q & (kRV - 1));
    mbar_expect_tx(bar, vbytes);
    tma_vplane<3>(g, &tm.u, &tm.glo, &tm.ghi, true, true, v0 + 8u * VS * (q & (kRV - 1)), bar,
                  x0, y0, zz);
  };
  pdl_wait();
  halo_wait(h, zb == 0, ze >= g.nzl);
  if (t == 0) {
    // ghost planes arrived through generic peer stores (acquired in
    // halo_wait); order them before this thread's async-proxy reads
    fence_proxy_async();
    issue_edge(zb - 1);
    for (int i = 0; i < kTmaLA; ++i) {
      if (zb + i < ze) issue_comp(zb + i);
      else {
        issue_edge(ze);
        break;
      }
    }
  }
  if (t == (EMRKC_EVWARP1 ? 32 : 0)) skip = (*(volatile const unsigned long long*)a.event) < level_floor(a.code_base, a.j, a.m, a.k);
  __syncthreads();
  if (skip) {  // aborted earlier: drain the prologue copies, release the neighbours
    const int np = 1 + min(kTmaLA, ze - zb) + (ze - zb < kTmaLA ? 1 : 0);
    for (int q = 0; q < np; ++q) mbar_wait(b0 + 8u * q, 0);
    halo_signal(h, zb == 0, ze >= g.nzl);
    return;
  }
  // per-row cells: V-box cell, mirrored neighbours, global column, validity
  constexpr int HXT = T::HX;
  const int cx = x0 + tx;
  const int dxm = cx > 0 ? -1 : 1, dxp = cx < g.n0 - 1 ? 1 : -1;
  int cell[R], dym[R], dyp[R];
  long long ipr[R];
  unsigned vmask = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int ry = ty + 4 * r, cy = y0 + ry;
    cell[r] = (ry + 1) * HXT + tx + 2;
    dym[r] = cy > 0 ? -HXT : HXT;
    dyp[r] = cy < g.n1 - 1 ? HXT : -HXT;
    const bool valid = cx < g.n0 && cy < g.n1;
    if (valid) vmask |= 1u << r;
    ipr[r] = valid ? (long long)cx + (long long)g.n0 * cy : 0;
  }
  bool bad_in = false, bad_out = false, guard = false;
  mbar_wait(b0, 0);
  mbar_wait(b0 + 8u, 0);
  for (int z = zb; z < ze; ++z) {
    const int p = z - zb + 1;
    if (t == 0) {
      if (z + kTmaLA < ze) issue_comp(z + kTmaLA);
      else if (z + kTmaLA == ze) issue_edge(ze);
    }
    mbar_wait(b0 + 8u * ((p + 1) & (kRV - 1)), ((p + 1) >> 3) & 1);
    const double* V0 = vst + (p & (kRV - 1)) * VS;
    const double* Vm = vst + ((p - 1) & (kRV - 1)) * VS;
    const double* Vp = vst + ((p + 1) & (kRV - 1)) * VS;
    const double* C0 = cst + ((z - zb) & (kRG - 1)) * T::CS * nb + t;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int c = cell[r];
      const double vc = V0[c];
      double D = fma(g.wc, vc, g.w[2] * (Vm[c] + Vp[c]));
      D = fma(g.w[0], V0[c + dxm] + V0[c + dxp], D);
      D = fma(g.w[1], V0[c + dym[r]] + V0[c + dyp[r]], D);
      const double* Cr = C0 + r * T::NT;  // row r of the tile: cells t + 128 r
      const double base = has2 ? fma(a.nu, vc, a.kappa * Cr[T::CS * f_um2]) : a.nu * vc;
      const double d1 = d1_is_u ? vc : Cr[0];
      const double dk = fma(a.mueta, fma(d1, a.inv_mue1, D), base);
      if (vmask >> r & 1u) {
        const long long i = ipr[r] + plane * z;
        bad_in |= !finite_hi(dk);
        double vput = dk;
        if (!LAST) {
          a.uk[i] = dk;
        } else {
          const double gv = Cr[T::CS * f_g1];
          const double bb = FIRST ? gv : fma(a.onu, gv, a.okappa * Cr[T::CS * (f_g1 + 1)]);
          const double o0 = fma(a.cG, dk, bb);
          a.outv[i] = o0;
          bad_out |= !finite_hi(o0);
          guard |= !(fabs(o0) <= 1e6);  // also a non-finite V
          vput = o0;
        }
        if (z == 0 && h.put_lo) h.put_lo[ipr[r]] = vput;
        if (z == g.nzl - 1 && h.put_hi) h.put_hi[ipr[r]] = vput;
      }
    }
    __syncthreads();
  }
  halo_signal(h, zb == 0, ze >= g.nzl);
  const unsigned long long base = a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1));
  if (bad_in) atomicMin(a.event, base + a.k);
  if (LAST && bad_out) atomicMin(a.event, base + a.m + 1);
  if (LAST && a.last && guard)
    atomicMin(a.event, a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
}

// ---------------------------------------------------------------------------
// k_vin_tb<K, FIRST>: inner stages k = 2 .. K+1 (= m) of outer stage j in one
// pass over HBM (temporal blocking of the V-only inner iteration).
//
// A block owns a 32 x 16 tile and a z-chunk [zb, ze) of the final stage and
// marches planes s. Its threads own the columns of the stage-2 region (the
// tile grown by K - 1 cells, x range widened to even cells), an x-adjacent
// PAIR of columns per thread, for the whole march. At step s
//   * d_1 of plane s arrives by TMA (box with an x halo of 4 and a y halo of
//     K, a 4-plane ring, two planes of look-ahead);
//   * stage k computes plane s - (k - 1); columns less than k - 2 cells
//     inside the region compute values nobody reads (no per-cell tests);
//   * the z neighbours and the centre of a column are the thread's own
//     values of the previous stage: each column keeps the last K + 1 planes
//     of d_1 and the last three planes of stages 2..K in registers, so a
//     stage reads only in-plane neighbours from shared memory — per pair two
//     128-bit loads (y - 1, y + 1) and two 64-bit loads (x - 1 of the left
//     cell, x + 1 of the right cell; the inner x neighbours are the pair's
//     own registers);
//   * stage k < m publishes its pair with one 128-bit store into a
//     double-buffered shared plane; stage k + 1 reads the plane published
//     one step earlier, so ONE __syncthreads per step orders every stage.
// The march is unrolled by the ring size: ring slot and buffer parity are
// compile-time constants and every shared access is [thread register +
// immediate]. Steps at the chunk ends (a stage outside its plane range, a z
// mirror, no d_1 plane left) take the EDGE instance with the tests.
// Stage K + 1 forms V of g_j = base + (mu_j dt / eta) d_m directly (V of
// g_{j-1}, g_{j-2} by 128-bit loads at the start of the step). Only d_1
// (plus its halo), V of g_{j-1}, g_{j-2} and V of g_j touch HBM: 24-32 B per
// node for all m - 1 stages instead of 16 + 32 (m - 3) + 40.
// Neumann mirror (P/src/monodomain.cpp:85-86): in x and y the per-thread
// neighbour addresses point at the mirrored cell; in z the column window is
// patched when a stage reaches plane 0 or nz - 1. Cells outside the grid
// hold values nobody reads. Recurrences exactly as k_vin_tma (increment
// form, same operation order: bitwise equal, tests/test_gpu_tb.py).
// ---------------------------------------------------------------------------
#ifndef EMRKC_TB_PIPE
#define EMRKC_TB_PIPE 0  // neighbour loads of stage k + 1 before stage k computes
#endif
constexpr int kTbRD = 4, kTbLA = 2;  // d_1 ring planes, look-ahead (RD >= LA + 2)
template <int K>
struct TbTile {
  static constexpr int TX = kTbTX, TY = kTbTY;
  static constexpr int HB = tb_hx(K);                         // x halo of the d_1 box (even)
  static constexpr int BX = TX + 2 * HB, BY = TY + 2 * K;     // d_1 box
  static constexpr int PS = BX * BY;
  static constexpr int PSS = (PS + 15) & ~15;                 // plane stride (128 B)
  // The region the threads own spans the whole box width (columns further
  // than K - 1 from the tile compute values nobody reads), so a thread's
  // shared address is linear in its index: 128-bit accesses of a warp never
  // conflict.
  static constexpr int PR = BX / 2;                           // column pairs per row
  static constexpr int RY = TY + 2 * (K - 1);                 // region rows
  static constexpr int NC = PR * RY;                          // threads owning pairs
  static constexpr int NT = (NC + 31) & ~31;
  // shared planes: d_1 ring, then two planes per published stage 2..K
  __host__ __device__ static constexpr int ring_off(int slot) { return 8 * slot * PSS; }
  __host__ __device__ static constexpr int stage_off(int k, int par) {
    return 8 * (kTbRD + 2 * (k - 2) + par) * PSS;
  }
  __host__ __device__ static constexpr int total() { return (kTbRD + 2 * (K - 1)) * PSS; }
};
static_assert(kTbRD == 4 && kTbRD >= kTbLA + 2, "k_vin_tb d_1 ring (march unrolled by 4)");
static_assert(kTbTY % 2 == 0 && tb_hx(kTbMaxK) >= kTbMaxK, "k_vin_tb tile");

template <int K>
constexpr size_t tb_smem_bytes() { return sizeof(double) * TbTile<K>::total() + 128; }
template <int K>
constexpr int tb_min_blocks() { return K == 1 ? 4 : (K == 2 ? 3 : (K == 3 ? 2 : 1)); }

// Compile-time loop: f(integral_constant<int, i>) for i in [B, E).
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// Shared-memory accesses at [register + immediate] (OFF >= 0) or, in the EDGE
// instance, [register + run-time offset] (the compiler cannot reorder them
// across the step barrier: volatile + memory clobber).
template <int OFF>
__device__ __forceinline__ void lds2(unsigned a, int off, double& x, double& y) {
  if constexpr (OFF >= 0)
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(x), "=d"(y) : "r"(a), "n"(OFF) : "memory");
  else
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a + off) : "memory");
}
template <int OFF>
__device__ __forceinline__ double lds1(unsigned a, int off) {
  double x;
  if constexpr (OFF >= 0)
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(x) : "r"(a), "n"(OFF) : "memory");
  else
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(a + off) : "memory");
  return x;
}
template <int OFF>
__device__ __forceinline__ void sts2(unsigned a, int off, double x, double y) {
  if constexpr (OFF >= 0)
    asm volatile("st.shared.v2.f64 [%0+%1], {%2, %3};" ::"r"(a), "n"(OFF), "d"(x), "d"(y) : "memory");
  else
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a + off), "d"(x), "d"(y) : "memory");
}
// all-ones accumulator of non-finite high words: max over (hi & sel) | 0x800fffff
__device__ __forceinline__ unsigned nf_acc(unsigned acc, double v, unsigned sel) {
  return max(acc, ((unsigned)__double2hiint(v) & sel) | 0x800fffffu);
}

// Per-thread constants and march state of k_vin_tb.
struct TbCtx {
  unsigned aC, aXm, aXp, aYm, aYp;  // shared byte addresses in plane 0
  unsigned b0, sel;
  bool own, gl, gh;
  int zb, ze, nz, lo1, hi1;
  long long plane;
  double inv_mue1;
};
template <int K>
struct TbState {
  // column windows: D[c][i] = d_1 at plane s - (DW - 1) + i; W[c][k - 2][i] =
  // stage k at plane (s - k + 1) - 2 + i, k = 2..K
  static constexpr int DW = K + 1 > 3 ? K + 1 : 3;  // d_1 planes kept per column
  double D[2][DW], W[2][K > 1 ? K - 1 : 1][3];
  unsigned acc[K + 2];  // per stage: all ones once an owned value was non-finite
  unsigned acc_o;
  bool guard;
  long long go;         // final-stage output offset of the step
  double2 v1n, v2n;     // V of g_{j-1} / g_{j-2} of the NEXT step's output plane (prefetched)
};

// One march step at ring phase (s - lo1) & 3 (PH, compile time, when
// !EDGE). EDGE = false is the steady state: every stage on a plane of the
// chunk, no z mirror, d_1 of plane s exists.
template <int K, int FIRST, bool EDGE, int PH>
__device__ __forceinline__ void tb_step(const Geom& g, const Halo& h, const TbArgs& a,
                                        const TbCtx& c, TbState<K>& st, const int s) {
  using T = TbTile<K>;
  constexpr int M = K + 1;
  constexpr int DW = TbState<K>::DW;
  const int i = s - c.lo1;
  const int ph = EDGE ? (i & 3) : PH;
  // V of g_{j-1} / g_{j-2} for the final stage's plane: loaded one step ahead
  // (under load the global-load latency exceeds a step; K = 2: +3%, K = 4:
  // +11%), except for K = 3, whose 72-register budget (two blocks per SM)
  // has no room for the carried values (spills: -10%) and loads them at the
  // start of the step they are used in.
  const int qo = s - K;
  double2 v1, v2;
  if constexpr (K != 3) {
    v1 = st.v1n;
    v2 = st.v2n;
    if (c.own && qo + 1 >= c.zb && qo + 1 < c.ze) {
      st.v1n = __ldg(reinterpret_cast<const double2*>(a.g1v + st.go + c.plane));
      if (!FIRST) st.v2n = __ldg(reinterpret_cast<const double2*>(a.g2v + st.go + c.plane));
    }
  } else {
    v1 = v2 = make_double2(0.0, 0.0);
    if (c.own && (!EDGE || (qo >= c.zb && qo < c.ze))) {
      v1 = __ldg(reinterpret_cast<const double2*>(a.g1v + st.go));
      if (!FIRST) v2 = __ldg(reinterpret_cast<const double2*>(a.g2v + st.go));
    }
  }
  const bool has_d = !EDGE || s < c.hi1;
  if (has_d) mbar_wait(c.b0 + 8u * ph, (i >> 2) & 1);
#pragma unroll
  for (int cc = 0; cc < 2; ++cc)
#pragma unroll
    for (int q = 0; q < DW - 1; ++q) st.D[cc][q] = st.D[cc][q + 1];
  if (has_d)
    lds2<EDGE ? -1 : T::ring_off(PH)>(c.aC, T::ring_off(1) * ph, st.D[0][DW - 1], st.D[1][DW - 1]);
  // In-plane neighbours of stage k: d_1 of plane s - 1 (k = 2) or the plane
  // stage k - 1 published one step ago. The loads of stage k + 1 are issued
  // before stage k computes (every plane read here was published before the
  // step's barrier), so their latency hides behind the arithmetic.
  double nb[2][6];  // ym0, ym1, yp0, yp1, xm0, xp1 (double-buffered by stage parity)
  auto load_nb = [&](auto kc) {
    constexpr int k = decltype(kc)::value;
    if constexpr (k <= M) {
      constexpr int SRC = EDGE ? -1
                               : (k == 2 ? T::ring_off((PH + 3) & 3)
                                         : T::stage_off(k >= 3 ? k - 1 : 2, (PH & 1) ^ 1));
      const int src = k == 2 ? T::ring_off(1) * ((ph + 3) & 3)
                             : T::stage_off(k >= 3 ? k - 1 : 2, 0) + T::ring_off(1) * ((ph & 1) ^ 1);
      double* n = nb[k & 1];
      lds2<SRC>(c.aYm, src, n[0], n[1]);
      lds2<SRC>(c.aYp, src, n[2], n[3]);
      n[4] = lds1<SRC>(c.aXm, src);
      n[5] = lds1<SRC>(c.aXp, src);
    }
  };
  if (EMRKC_TB_PIPE) load_nb(std::integral_constant<int, 2>{});
  static_for<2, M + 1>([&](auto kc) {
    constexpr int k = decltype(kc)::value;
    constexpr int hk = K + 1 - k;
    const int q = s - (k - 1);
    const bool active = !EDGE || (q >= (c.gl ? c.zb - hk : max(0, c.zb - hk)) &&
                                  q < (c.gh ? c.ze + hk : min(c.nz, c.ze + hk)));
    const bool mlo = EDGE && q < 1 && !c.gl, mhi = EDGE && q + 1 >= c.nz && !c.gh;
    const bool own_plane = !EDGE || (q >= c.zb && q < c.ze);
    const double mueta = a.mueta[k], nu = a.nu[k], kappa = a.kappa[k];
    if (EMRKC_TB_PIPE) load_nb(std::integral_constant<int, k + 1>{});
    else load_nb(kc);
    const double* n = nb[k & 1];
    double dk[2] = {0.0, 0.0};
    if (active) {
      double z0[2], z1[2], z2[2];
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        if constexpr (k == 2) {
          z0[cc] = st.D[cc][DW - 3];
          z1[cc] = st.D[cc][DW - 2];
          z2[cc] = st.D[cc][DW - 1];
        } else {
          z0[cc] = st.W[cc][k - 3][0];
          z1[cc] = st.W[cc][k - 3][1];
          z2[cc] = st.W[cc][k - 3][2];
        }
        if (mlo) z0[cc] = z2[cc];
        if (mhi) z2[cc] = z0[cc];
      }
      const double xs[2] = {n[4] + z1[1], z1[0] + n[5]};
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const double vc = z1[cc];
        double L = fma(g.wc, vc, g.w[2] * (z0[cc] + z2[cc]));
        L = fma(g.w[0], xs[cc], L);
        L = fma(g.w[1], n[cc] + n[2 + cc], L);
        const double d1c = st.D[cc][DW - k];
        double bs = nu * vc;
        if constexpr (k == 3) bs = fma(nu, vc, kappa * d1c);
        if constexpr (k >= 4) bs = fma(nu, vc, kappa * st.W[cc][k >= 4 ? k - 4 : 0][0]);
        dk[cc] = fma(mueta, fma(d1c, c.inv_mue1, L), bs);
        if (own_plane) st.acc[k] = nf_acc(st.acc[k], dk[cc], c.sel);
      }
      if constexpr (k < M) {
        sts2<EDGE ? -1 : T::stage_off(k < M ? k : 2, PH & 1)>(
            c.aC, T::stage_off(k < M ? k : 2, 0) + T::ring_off(1) * (ph & 1), dk[0], dk[1]);
      } else if (c.own && own_plane) {
        // final stage: V of g_j
        double2 o;
        o.x = fma(a.cG, dk[0], FIRST ? v1.x : fma(a.onu, v1.x, a.okappa * v2.x));
        o.y = fma(a.cG, dk[1], FIRST ? v1.y : fma(a.onu, v1.y, a.okappa * v2.y));
        *reinterpret_cast<double2*>(a.outv + st.go) = o;
        if (EDGE) {
          if (q == 0 && h.put_lo) *reinterpret_cast<double2*>(h.put_lo + (st.go - c.plane * q)) = o;
          if (q == c.nz - 1 && h.put_hi)
            *reinterpret_cast<double2*>(h.put_hi + (st.go - c.plane * q)) = o;
        }
        st.acc_o = nf_acc(nf_acc(st.acc_o, o.x, 0xffffffffu), o.y, 0xffffffffu);
        st.guard |= !(fabs(o.x) <= 1e6) || !(fabs(o.y) <= 1e6);  // also a non-finite V
      }
    }
    if constexpr (k < M) {  // the stage's own windows move every step
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        st.W[cc][k < M ? k - 2 : 0][0] = st.W[cc][k < M ? k - 2 : 0][1];
        st.W[cc][k < M ? k - 2 : 0][1] = st.W[cc][k < M ? k - 2 : 0][2];
        st.W[cc][k < M ? k - 2 : 0][2] = dk[cc];
      }
    }
  });
  st.go += c.plane;
}

template <int K, int FIRST>
__global__ void __launch_bounds__(TbTile<K>::NT, tb_min_blocks<K>())
    k_vin_tb(const Geom g, const Halo h, const TbArgs a, const __grid_constant__ TmaTb tm) {
  using T = TbTile<K>;
  constexpr int M = K + 1;  // m
  constexpr int PSS = T::PSS, BX = T::BX;
  extern __shared__ __align__(128) double smem_tma[];
  double* sm = smem_tma + ((128u - (smem_u32(smem_tma) & 127u)) & 127u) / 8;
  __shared__ __align__(8) unsigned long long bars[kTbRD];
  __shared__ int skip;
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * T::TX, y0 = blockIdx.y * T::TY;
  const int zb = blockIdx.z * a.zc;
  const int ze = min(g.nzl, zb + a.zc);
  const int n0 = g.n0, n1 = g.n1, nz = g.nzl;
  pdl_launch_dependents();
  if (t == 0) {
    for (int s = 0; s < kTbRD; ++s) mbar_init(smem_u32(&bars[s]), 1);
    mbar_fence_init();
    prefetch_tensormap(&tm.d1);
  }
  __syncthreads();
  pdl_wait();
  // slab faces with a neighbour (h.lo / h.hi: its K d_1 ghost planes) march
  // into the ghosts; global boundaries mirror (P/src/monodomain.cpp:85-86)
  const bool gl = h.lo != nullptr, gh = h.hi != nullptr;
  const int lo1 = max(gl ? -K : 0, zb - K), hi1 = min(gh ? nz + K : nz, ze + K);  // d_1 planes
  const int tlast = ze - 1 + K;                           // last step
  const unsigned b0 = smem_u32(bars), dbase = smem_u32(sm);
  auto issue = [&](int s) {  // thread 0: d_1 of plane s in [lo1, hi1)
    const int i = s - lo1;
    const unsigned bar = b0 + 8u * (i & (kTbRD - 1));
    mbar_expect_tx(bar, 8u * T::PS);
    const unsigned dd = dbase + 8u * PSS * (i & (kTbRD - 1));
    if (s < 0) tma_load_3d(dd, &tm.d1lo, bar, x0 - T::HB, y0 - K, s + K);
    else if (s >= nz) tma_load_3d(dd, &tm.d1hi, bar, x0 - T::HB, y0 - K, s - nz);
    else tma_load_3d(dd, &tm.d1, bar, x0 - T::HB, y0 - K, s);
  };
  const int npro = min(kTbLA, hi1 - lo1);
  if (t == 0) {
    if (lo1 < 0 || hi1 > nz) {
      halo_wait(h, lo1 < 0, hi1 > nz);
      fence_proxy_async();  // peer-stored ghosts before the async-proxy reads
    }
    for (int i = 0; i < npro; ++i) issue(lo1 + i);
    skip = (*(volatile const unsigned long long*)a.event) < level_floor(a.code_base, a.j, a.m, 2);
  }
  __syncthreads();
  if (skip) {
    for (int i = 0; i < npro; ++i) mbar_wait(b0 + 8u * i, 0);
    halo_signal(h, zb == 0, ze >= nz);  // release the neighbours
    return;
  }
  // The thread's pair of columns (cells 0 and 1, x-adjacent, even x first):
  // shared byte addresses of the pair and of its mirrored in-plane
  // neighbours inside plane 0 (a plane's offset is an immediate), ownership
  // (the pair lies in the tile and the grid) and the output offset. Threads
  // past the last pair repeat an earlier pair (identical values, no outputs).
  const int tt = t < T::NC ? t : t - T::NC;
  const int px = tt % T::PR, cy = tt / T::PR;
  const int gx = x0 - T::HB + 2 * px, gy = y0 - (K - 1) + cy;
  const int ci = BX + 2 * tt;  // cell 0 in the box: row cy + 1, column 2 px
  TbCtx c;
  c.own = t < T::NC && gx >= x0 && gx < min(x0 + T::TX, n0) && gy >= y0 &&
          gy < min(y0 + T::TY, n1);
  c.sel = c.own ? 0xffffffffu : 0u;
  c.aC = dbase + 8u * ci;
  // x - 1 of cell 0 (mirror at x = 0; box column 0 has no left cell: any value)
  c.aXm = c.aC + ((gx > 0 && px > 0) ? -8 : 8);
  // x + 1 of cell 1 (mirror at x = n0 - 1; none right of the last box column)
  c.aXp = c.aC + 8u + ((gx + 1 < n0 - 1 && px < T::PR - 1) ? 8 : -8);
  c.aYm = c.aC + (gy > 0 ? -8 * BX : 8 * BX);
  c.aYp = c.aC + (gy < n1 - 1 ? 8 * BX : -8 * BX);
  c.b0 = b0;
  c.gl = gl;
  c.gh = gh;
  c.zb = zb;
  c.ze = ze;
  c.nz = nz;
  c.lo1 = lo1;
  c.hi1 = hi1;
  c.plane = g.plane;
  c.inv_mue1 = a.inv_mue1;
  TbState<K> st;
  st.go = (long long)gx + (long long)n0 * gy + g.plane * (lo1 - K);
#pragma unroll
  for (int k = 0; k <= M; ++k) st.acc[k] = 0u;
  st.acc_o = 0u;
  st.guard = false;
  st.v1n = st.v2n = make_double2(0.0, 0.0);
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
#pragma unroll
    for (int q = 0; q < TbState<K>::DW; ++q) st.D[cc][q] = 0.0;
#pragma unroll
    for (int k = 0; k < K - 1; ++k) st.W[cc][k][0] = st.W[cc][k][1] = st.W[cc][k][2] = 0.0;
  }
  // steady steps: every stage's plane s - k + 1 lies in [max(zb, 1), min(ze, nz - 1))
  const int st0 = max(zb, 1) + K, st1 = min(ze, nz - 1);
  int s = lo1;
  // edge steps up to the first steady step at ring phase 0
  for (; s <= tlast && (s < st0 || ((s - lo1) & 3) != 0); ++s) {
    if (t == 0 && s + kTbLA < hi1) issue(s + kTbLA);
    tb_step<K, FIRST, true, 0>(g, h, a, c, st, s);
    __syncthreads();
  }
  for (; s + 3 <= st1; s += 4) {
    if (t == 0 && s + kTbLA < hi1) issue(s + kTbLA);
    tb_step<K, FIRST, false, 0>(g, h, a, c, st, s);
    __syncthreads();
    if (t == 0 && s + 1 + kTbLA < hi1) issue(s + 1 + kTbLA);
    tb_step<K, FIRST, false, 1>(g, h, a, c, st, s + 1);
    __syncthreads();
    if (t == 0 && s + 2 + kTbLA < hi1) issue(s + 2 + kTbLA);
    tb_step<K, FIRST, false, 2>(g, h, a, c, st, s + 2);
    __syncthreads();
    if (t == 0 && s + 3 + kTbLA < hi1) issue(s + 3 + kTbLA);
    tb_step<K, FIRST, false, 3>(g, h, a, c, st, s + 3);
    __syncthreads();
  }
  for (; s <= tlast; ++s) {
    if (t == 0 && s + kTbLA < hi1) issue(s + kTbLA);
    tb_step<K, FIRST, true, 0>(g, h, a, c, st, s);
    __syncthreads();
  }
  halo_signal(h, zb == 0, ze >= nz);
  const unsigned long long base = a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1));
  unsigned badk = 0u;
#pragma unroll
  for (int k = 2; k <= M; ++k)
    if (st.acc[k] == 0xffffffffu) badk |= 1u << k;
  if (badk) atomicMin(a.event, base + (unsigned long long)(__ffs(badk) - 1));
  if (st.acc_o == 0xffffffffu) atomicMin(a.event, base + a.m + 1);
  if (a.last && st.guard)
    atomicMin(a.event, a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
}

// ---------------------------------------------------------------------------
// V-only inner stage k >= 2 (LAST: k == m, forms V of g_j).
// ---------------------------------------------------------------------------
template <int DIM, int LAST, int FIRST>
__global__ void __launch_bounds__(kFThreads)
    k_vin_fast(const Geom g, const Halo h, const FastInnerArgs a) {
  const int bz0 = (DIM == 3 ? blockIdx.z * a.zc : blockIdx.y * FBY * a.zc);
  const int bz1 = (DIM == 3 ? bz0 + a.zc : bz0 + FBY * a.zc);
  halo_wait(h, bz0 == 0, bz1 >= g.nzl);
  if (prologue(a.event, level_floor(a.code_base, a.j, a.m, a.k), nullptr)) {  // aborted earlier: still release the neighbours
    halo_signal(h, bz0 == 0, bz1 >= g.nzl);
    return;
  }
  const Col<DIM> c = col_here<DIM>(g, a.zc);
  bool bad_in = false, bad_out = false, guard = false;
  if (c.valid) {
    const double* __restrict__ U = a.um1;
    const Nbr<DIM> o = nbr_of<DIM>(g, c);
    double vm = zval(U, g, c.ip, c.z0 - 1, h.lo, h.hi);
    double vc = zval(U, g, c.ip, c.z0, h.lo, h.hi);
    for (int z = c.z0; z < c.z1; ++z) {
      const double vp = zval(U, g, c.ip, z + 1, h.lo, h.hi);
      const long long i = c.ip + g.plane * z;
      const double D = lap_fast<DIM>(g, U, i, o, vm, vc, vp);
      const double d1 = __ldg(a.d1 + i);
      const double base = a.um2 ? fma(a.nu, vc, a.kappa * __ldg(a.um2 + i)) : a.nu * vc;
      const double dk = fma(a.mueta, fma(d1, a.inv_mue1, D), base);
      bad_in |= !finite_hi(dk);
      double vput = dk;
      if (!LAST) {
        a.uk[i] = dk;
      } else {
        const double gv = __ldg(a.g1v + i);
        const double b0 = FIRST ? gv : fma(a.onu, gv, a.okappa * __ldg(a.g2v + i));
        const double o0 = fma(a.cG, dk, b0);
        a.outv[i] = o0;
        bad_out |= !finite_hi(o0);
        guard |= !(fabs(o0) <= 1e6);  // also a non-finite V
        vput = o0;
      }
      if (z == 0 && h.put_lo) h.put_lo[c.ip] = vput;
      if (z == g.nzl - 1 && h.put_hi) h.put_hi[c.ip] = vput;
      vm = vc;
      vc = vp;
    }
  }
  const unsigned long long base = a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1));
  if (bad_in) atomicMin(a.event, base + a.k);
  if (LAST && bad_out) atomicMin(a.event, base + a.m + 1);
  if (LAST && a.last && guard)
    atomicMin(a.event, a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
  halo_signal(h, bz0 == 0, bz1 >= g.nzl);
}

template <int DIM>
dim3 fgrid(const Geom& g, int zc) {
  if (DIM == 3)
    return dim3((g.n0 + FBX - 1) / FBX, (g.n1 + FBY - 1) / FBY, (g.nzl + zc - 1) / zc);
  if (DIM == 2) {
    const int chunks = (g.nzl + zc - 1) / zc;
    return dim3((g.n0 + FBX - 1) / FBX, (chunks + FBY - 1) / FBY, 1);
  }
  return dim3((g.nzl + kFThreads - 1) / kFThreads, 1, 1);
}

#if EMRKC_EXPERIMENTAL  // k_fused2: measured slower than the two-kernel step
// ---------------------------------------------------------------------------
// k_fused2: a whole emRKC step with s = 1, m = 2 in ONE pass over HBM (3-D,
// whole grid): the node update (exponential Euler of the gates, f_S(y_E),
// 7-point stencil, inner stage 1 -> d_1, gate rows of g_1) of plane z and
// inner stage 2 + the outer update of plane z - 1 (V of g_1), so d_1 never
// touches HBM: 64 B per node instead of 64 (node kernel) + 24 (inner
// kernel). Inner stage 2 needs f_F(d_1) on the x/y neighbours of a tile,
// which other blocks compute: the grid is persistent and co-resident (a
// cooperative launch, one 64 x ~14 column tile and a z-range per block, two
// blocks per SM), each block stores the edge rows / columns of its d_1
// plane into an L2-resident exchange ring and publishes the plane on a
// monotone flag (fence + relaxed store); iteration z runs inner stage 2 of
// plane z - 2 first (the neighbours published its edges one whole
// iteration earlier: lanes 0..3 poll one flag each, then fence, then the
// edges are read with ld.cg) and then the node update of plane z. The stencil has no order-dependent
// reductions: the arithmetic is k_node_tma<3,1,1>'s and k_vin_tma_r<1,1>'s
// operation for operation (bitwise equal to the two-kernel step).
// Per block: V boxes (68 x 16) two planes ahead, gate boxes (64 x 14 x 3)
// one plane ahead (TMA), a 3-plane ring of d_1 tiles with a one-cell halo
// filled from the neighbours' edges (or mirrored at the grid boundary,
// P/src/monodomain.cpp:85-86), z-chunks recompute d_1 one plane beyond
// each end. Nodes outside the fast ionic window take the reference-order
// path in a per-plane second pass (rare).
// ---------------------------------------------------------------------------
constexpr int kFuRV = 4, kFuRG = 2, kFuRD = 3, kFuRX = 4;
constexpr int kFuVX = kFuTX + 4, kFuVY = kFuTY + 2;
constexpr int kFuVS = ((kFuVX * kFuVY) + 15) & ~15;
constexpr int kFuGF = kFuTX * kFuTY;  // one gate field of a tile
constexpr int kFuGS = 3 * kFuGF;
constexpr int kFuDX = kFuTX + 2;
constexpr int kFuDS = ((kFuDX * (kFuTY + 2)) + 15) & ~15;
static_assert(kFuTX == 64 && kFuNT == 256 && kFuTY * kFuTX <= 4 * kFuNT, "fused tile");

constexpr size_t fused_smem_bytes() {
  return sizeof(double) * (kFuRV * kFuVS + kFuRG * kFuGS + kFuRD * kFuDS) + 128;
}

__device__ __forceinline__ void st_relaxed_gpu_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kFuNT, 2)
    k_fused2(const Geom g, const FusedArgs A, const __grid_constant__ TmaFused tm) {
  const FastArgs& a = A.f;
  extern __shared__ __align__(128) double smem_fu[];
  double* vst = smem_fu + ((128u - (smem_u32(smem_fu) & 127u)) & 127u) / 8;  // [RV][VS]
  double* gst = vst + kFuRV * kFuVS;                                          // [RG][GS]
  double* dst = gst + kFuRG * kFuGS;                                          // [RD][DS]
  __shared__ double tab[256];
  __shared__ __align__(8) unsigned long long vbar[kFuRV], gbar[kFuRG];
  __shared__ int skip, timed_out;
  __shared__ unsigned long long rlo[kFuNT / 32], rhi[kFuNT / 32];
  const int t = threadIdx.x;
  const int ntile = A.ntx * A.nty;
  const int zi = blockIdx.x / ntile, tile = blockIdx.x % ntile;
  const int txi = tile % A.ntx, tyi = tile / A.ntx;
  const int x0 = txi * kFuTX;
  const int y0 = (int)((long long)tyi * g.n1 / A.nty);
  const int TYH = (int)((long long)(tyi + 1) * g.n1 / A.nty) - y0;
  const int nz = g.nzl;
  const int zb = (int)((long long)zi * nz / A.nzc), ze = (int)((long long)(zi + 1) * nz / A.nzc);
  const int zA = max(zb - 1, 0), zE = min(ze + 1, nz);  // d_1 planes [zA, zE)
  const long long nn = g.nn, plane = g.plane;
  if (t == 0) {
    for (int q = 0; q < kFuRV; ++q) mbar_init(smem_u32(&vbar[q]), 1);
    for (int q = 0; q < kFuRG; ++q) mbar_init(smem_u32(&gbar[q]), 1);
    mbar_fence_init();
    prefetch_tensormap(&tm.v);
    prefetch_tensormap(&tm.gates);
    skip = (*(volatile const unsigned long long*)a.event) < level_floor(a.code_base, a.j, a.m, 1);
    timed_out = 0;
  }
  load_exp_table(tab, t, kFuNT);
  __syncthreads();
  // every block takes the same decision: events of this launch are >= the floor
  if (skip) return;
  const unsigned v0s = smem_u32(vst), g0s = smem_u32(gst);
  auto issue_v = [&](int zz) {  // V box of plane zz in [zA - 1, zE]
    const int q = zz - zA + 1;
    const unsigned bar = smem_u32(&vbar[q & (kFuRV - 1)]);
    mbar_expect_tx(bar, 8u * kFuVX * kFuVY);
    tma_vplane<3>(g, &tm.v, nullptr, nullptr, false, false,
                  v0s + 8u * kFuVS * (q & (kFuRV - 1)), bar, x0, y0, zz);
  };
  auto issue_g = [&](int zz) {  // gate box of plane zz in [zA, zE)
    const int q = zz - zA;
    const unsigned bar = smem_u32(&gbar[q & (kFuRG - 1)]);
    mbar_expect_tx(bar, 8u * kFuGS);
    tma_load_4d(g0s + 8u * kFuGS * (q & (kFuRG - 1)), &tm.gates, bar, x0, y0, zz, 1);
  };
  if (t == 0) {
    issue_v(zA - 1);
    issue_v(zA);
    if (zA + 1 <= zE) issue_v(zA + 1);
    issue_g(zA);
  }
  const int lx = t & (kFuTX - 1), ly0 = t / kFuTX;
  const int cx = x0 + lx;
  const int dxm = cx > 0 ? -1 : 1, dxp = cx < g.n0 - 1 ? 1 : -1;
  const bool stx = cx >= g.st_lo[0] && cx <= g.st_hi[0];
  double* const outv = a.out;  // V block of g_1 (stage 2); gate rows at + nn
  unsigned finacc = 0x7ff00000u;
  bool bad_slow = false, bad_in = false, bad_out = false, guard = false, any_out = false;
  double glo = 2.0, ghi = -1.0;
  mbar_wait(smem_u32(&vbar[0]), 0);  // V(zA - 1)
  mbar_wait(smem_u32(&vbar[1]), 0);  // V(zA)
  const int base_cta = zi * ntile;
  // neighbour of side s (W, E, S, N) in this z-chunk, -1 at the grid edge
  const int nbr = t < 4 ? (t == 0 ? (txi > 0 ? tile - 1 : -1)
                                  : t == 1 ? (txi < A.ntx - 1 ? tile + 1 : -1)
                                  : t == 2 ? (tyi > 0 ? tile - A.ntx : -1)
                                           : (tyi < A.nty - 1 ? tile + A.ntx : -1))
                        : -1;
  // Iteration z: phase B of plane z - 2 (its d_1 edges were published by the
  // neighbours one whole iteration ago), then phase A of plane z.
  for (int z = zA; z <= ze + 1; ++z) {
    const int zz = z - 2;
    const bool doB = zz >= zb && zz < ze;
    // ---- phase B: inner stage 2 + outer update of plane zz
    if (doB) {
      if (nbr >= 0) {  // lanes 0..3 of warp 0: one neighbour flag each
        const unsigned long long want = A.epoch + (unsigned long long)(zz + 1);
        const unsigned long long t0 = globaltimer_ns();
        while (ld_relaxed_gpu_u64(A.flags + base_cta + nbr) < want) {
          if (globaltimer_ns() - t0 > 4000000000ull) {  // a neighbour never came: bail
            timed_out = 1;
            atomicMin(a.event, 0ull);
            break;
          }
        }
        fence_acq_rel_gpu();
      }
      __syncthreads();
      if (timed_out) return;
      double* Dz = dst + (zz % kFuRD) * kFuDS;
      const int slot = zz & (kFuRX - 1);
      auto xedge = [&](int nbtile, int side, int i) {
        return __ldcg(A.xch + ((size_t)(base_cta + nbtile) * kFuRX + slot) * 4 * kFuTX +
                      side * kFuTX + i);
      };
      if (t < kFuTY) {  // west halo column <- the west tile's east edge (or mirror x = 1)
        if (t < TYH)
          Dz[(t + 1) * kFuDX] = txi > 0 ? xedge(tile - 1, 1, t) : Dz[(t + 1) * kFuDX + 2];
      } else if (t >= 64 && t < 64 + kFuTY) {  // east <- east tile's west edge (or x = n0 - 2)
        const int i = t - 64;
        if (i < TYH)
          Dz[(i + 1) * kFuDX + kFuTX + 1] =
              txi < A.ntx - 1 ? xedge(tile + 1, 0, i) : Dz[(i + 1) * kFuDX + kFuTX - 1];
      } else if (t >= 128 && t < 192) {  // south <- south tile's north edge (or y = 1)
        const int i = t - 128;
        Dz[i + 1] = tyi > 0 ? xedge(tile - A.ntx, 3, i) : Dz[2 * kFuDX + i + 1];
      } else if (t >= 192) {  // north <- north tile's south edge (or y = n1 - 2)
        const int i = t - 192;
        Dz[(TYH + 1) * kFuDX + i + 1] =
            tyi < A.nty - 1 ? xedge(tile + A.ntx, 2, i) : Dz[(TYH - 1) * kFuDX + i + 1];
      }
      __syncthreads();
      const double* Dm = dst + ((zz == 0 ? 1 : zz - 1) % kFuRD) * kFuDS;
      const double* Dp = dst + ((zz == nz - 1 ? nz - 2 : zz + 1) % kFuRD) * kFuDS;
      const double* Vg = vst + ((zz - zA + 1) & (kFuRV - 1)) * kFuVS;  // V of g_0 at zz
      for (int r = 0; r < 4; ++r) {
        const int ly = ly0 + 4 * r;
        if (ly >= TYH) break;
        const int c = (ly + 1) * kFuDX + lx + 1;
        const double d1 = Dz[c];
        double D = fma(g.wc, d1, g.w[2] * (Dm[c] + Dp[c]));
        D = fma(g.w[0], Dz[c - 1] + Dz[c + 1], D);
        D = fma(g.w[1], Dz[c - kFuDX] + Dz[c + kFuDX], D);
        const double dk = fma(A.mueta2, fma(d1, A.inv_mue1, D), A.nu2 * d1);
        const double o0 = fma(A.cG2, dk, Vg[(ly + 1) * kFuVX + lx + 2]);
        outv[(cx + (long long)g.n0 * (y0 + ly)) + plane * zz] = o0;
        bad_in |= !finite_hi(dk);
        bad_out |= !finite_hi(o0);
        guard |= !(fabs(o0) <= 1e6);  // also a non-finite V
      }
    }
    // V(zz) and d_1(zz - 1) are free: the ring slots take V(z + 2) and d_1(z)
    if (doB) __syncthreads();
    const bool doA = z < zE;
    const int qv = z - zA + 1;
    if (t == 0) {
      if (z + 2 <= zE) issue_v(z + 2);
      if (z + 1 < zE) issue_g(z + 1);
    }
    // ---- phase A: node update of plane z -> d_1 (smem + edges), gates of g_1
    unsigned slow = 0;
    if (doA) {
      mbar_wait(smem_u32(&vbar[(qv + 1) & (kFuRV - 1)]), ((qv + 1) >> 2) & 1);
      mbar_wait(smem_u32(&gbar[(z - zA) & (kFuRG - 1)]), ((z - zA) >> 1) & 1);
      const double* V0 = vst + (qv & (kFuRV - 1)) * kFuVS;
      const double* Vm = vst + ((qv - 1) & (kFuRV - 1)) * kFuVS;
      const double* Vp = vst + ((qv + 1) & (kFuRV - 1)) * kFuVS;
      const double* G0 = gst + ((z - zA) & (kFuRG - 1)) * kFuGS;
      double* D0 = dst + (z % kFuRD) * kFuDS;
      double* X = A.xch + ((size_t)blockIdx.x * kFuRX + (z & (kFuRX - 1))) * 4 * kFuTX;
      const bool outp = z >= zb && z < ze;
      const bool stz = stim_z<3>(g, z) && stx;
      for (int r = 0; r < 4; ++r) {
        const int ly = ly0 + 4 * r;
        if (ly >= TYH) break;
        const int cy = y0 + ly;
        const int c = (ly + 1) * kFuVX + lx + 2;
        const double vc = V0[c];
        if (!(fabs(vc - a.vmid) <= a.vfast)) {
          slow |= 1u << r;
          continue;
        }
        const double xs = V0[c + dxm] + V0[c + dxp];
        const double ys = V0[c + (cy > 0 ? -kFuVX : kFuVX)] + V0[c + (cy < g.n1 - 1 ? kFuVX : -kFuVX)];
        const int gi = ly * kFuTX + lx;
        NodeOut o = node_update_s<3, 1, 1, 0>(g, a, tab, Vm[c], vc, Vp[c], xs, ys, G0[gi],
                                             G0[kFuGF + gi], G0[2 * kFuGF + gi], 0.0, nullptr, 0);
        if (stz && cy >= g.st_lo[1] && cy <= g.st_hi[1]) o.o0 = fma(a.mue1, a.stim, o.o0);
        D0[(ly + 1) * kFuDX + lx + 1] = o.o0;
        if (lx == 0) X[ly] = o.o0;
        if (lx == kFuTX - 1) X[kFuTX + ly] = o.o0;
        if (ly == 0) X[2 * kFuTX + lx] = o.o0;
        if (ly == TYH - 1) X[3 * kFuTX + lx] = o.o0;
        if (outp) {
          double* po = a.out + (cx + (long long)g.n0 * cy) + plane * z;
          po[nn] = o.o1;
          po[2 * nn] = o.o2;
          po[3 * nn] = o.o3;
          finacc = min(finacc,
                       ~(unsigned)__double2hiint((o.o0 + o.o1) + (o.o2 + o.o3)) & 0x7ff00000u);
          any_out = true;
          if (a.last) {
            glo = o.o1 < glo ? o.o1 : glo;
            ghi = ghi < o.o1 ? o.o1 : ghi;
            glo = o.o2 < glo ? o.o2 : glo;
            ghi = ghi < o.o2 ? o.o2 : ghi;
            glo = o.o3 < glo ? o.o3 : glo;
            ghi = ghi < o.o3 ? o.o3 : ghi;
          }
        }
      }
    }
    // nodes outside the fast window: reference-order ionic path, this plane
    if (__syncthreads_or(slow != 0)) {
      if (slow) {
        const double* V0 = vst + (qv & (kFuRV - 1)) * kFuVS;
        const double* Vm = vst + ((qv - 1) & (kFuRV - 1)) * kFuVS;
        const double* Vp = vst + ((qv + 1) & (kFuRV - 1)) * kFuVS;
        const double* G0 = gst + ((z - zA) & (kFuRG - 1)) * kFuGS;
        double* D0 = dst + (z % kFuRD) * kFuDS;
        double* X = A.xch + ((size_t)blockIdx.x * kFuRX + (z & (kFuRX - 1))) * 4 * kFuTX;
        const bool outp = z >= zb && z < ze;
        const bool stz = stim_z<3>(g, z) && stx;
        for (int r = 0; r < 4; ++r) {
          if (!(slow >> r & 1u)) continue;
          const int ly = ly0 + 4 * r;
          const int cy = y0 + ly;
          const int c = (ly + 1) * kFuVX + lx + 2;
          const double xs = V0[c + dxm] + V0[c + dxp];
          const double ys =
              V0[c + (cy > 0 ? -kFuVX : kFuVX)] + V0[c + (cy < g.n1 - 1 ? kFuVX : -kFuVX)];
          const int gi = ly * kFuTX + lx;
          const double stim = (stz && cy >= g.st_lo[1] && cy <= g.st_hi[1]) ? a.stim : 0.0;
          double q[4] = {0.0, 0.0, 0.0, 0.0};
          const NodeOut o = node_update_s<3, 1, 1, 1>(g, a, tab, Vm[c], V0[c], Vp[c], xs, ys,
                                                      G0[gi], G0[kFuGF + gi], G0[2 * kFuGF + gi],
                                                      stim, q, 1);
          D0[(ly + 1) * kFuDX + lx + 1] = o.o0;
          if (lx == 0) X[ly] = o.o0;
          if (lx == kFuTX - 1) X[kFuTX + ly] = o.o0;
          if (ly == 0) X[2 * kFuTX + lx] = o.o0;
          if (ly == TYH - 1) X[3 * kFuTX + lx] = o.o0;
          if (outp) {
            double* po = a.out + (cx + (long long)g.n0 * cy) + plane * z;
            po[nn] = o.o1;
            po[2 * nn] = o.o2;
            po[3 * nn] = o.o3;
            bad_slow |= !finite_hi((o.o0 + o.o1) + (o.o2 + o.o3));
            any_out = true;
            if (a.last) {
              glo = fmin(glo, fmin(o.o1, fmin(o.o2, o.o3)));
              ghi = fmax(ghi, fmax(o.o1, fmax(o.o2, o.o3)));
            }
          }
        }
      }
      __syncthreads();
    }
    // publish d_1 plane z (its edges) to the neighbours
    if (t == 0 && doA) {
      __threadfence();
      st_relaxed_gpu_u64(A.flags + blockIdx.x, A.epoch + (unsigned long long)(z + 1));
    }
  }
  // ---- events (first failing check in program order wins), gate range
  const unsigned long long base = a.code_base + (unsigned long long)((a.j - 1) * (a.m + 1));
  if ((finacc == 0u || bad_slow) && !a.exex) {
    bool inner = false;
    for (int r = 0; r < 4; ++r) {
      const int ly = ly0 + 4 * r;
      if (ly >= TYH) break;
      Col<3> c;
      c.c0 = cx;
      c.c1 = y0 + ly;
      c.ip = cx + (long long)g.n0 * (y0 + ly);
      c.z0 = zb;
      c.z1 = ze;
      c.valid = true;
      inner |= inner_nonfinite<3>(g, Halo{}, a.g1, c, nbr_of<3>(g, c), a.eta);
    }
    atomicMin(a.event, base + (inner ? 1ull : (unsigned long long)(a.m + 1)));
  }
  if (bad_in) atomicMin(a.event, base + 2ull);
  if (bad_out) atomicMin(a.event, base + (unsigned long long)(a.m + 1));
  if (a.last && guard)
    atomicMin(a.event, a.code_base + (unsigned long long)(a.s * (a.m + 1) + 1));
  if (a.last) {
    unsigned long long lo = any_out ? ord_of(glo) : ~0ull, hi = any_out ? ord_of(ghi) : 0ull;
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((t & 31) == 0) {
      rlo[t >> 5] = lo;
      rhi[t >> 5] = hi;
    }
    __syncthreads();
    if (t == 0) {
      for (int w = 1; w < kFuNT / 32; ++w) {
        lo = min(lo, rlo[w]);
        hi = max(hi, rhi[w]);
      }
      if (lo != ~0ull) atomicMin(a.gate_slot, lo);
      if (hi != 0ull) atomicMax(a.gate_slot + 1, hi);
    }
  }
}
#endif  // EMRKC_EXPERIMENTAL (k_fused2)

}  // namespace

// Planes per block (z-chunk length): 16 amortises the block prologue (abort
// word, exp table, the cp.async pipeline fill); halved while the grid would
// give fewer than ~2 waves of 148 SMs x 5 resident blocks.
// z-chunk of the staged 3-D node kernels. A launch of B = tiles x
// ceil(nz / zc) blocks on S resident slots takes about
//   W (1 + c0 / zc) + alpha (zc + c0),   W = tiles nz / S planes per slot:
// every block pays a prologue worth c0 planes (barrier init, table, pipeline
// fill), and the launch ends with a tail of about alpha blocks (the last
// slots run part-empty). Measured on B200 (gpurun_out/ab_pair_zc*.log:
// 128^3, 256x256x128, 512x512x256, sweep N = 100 / 200; r01 zc sweeps of
// k_node_tma): c0 / alpha = 3.75 planes for k_node_pair and 7.5 for
// k_node_tma (half the work per plane), i.e. zc* = sqrt(c0 W / alpha):
// 128^3 -> 8 / 13, 256x256x128 -> 14, 512x512x256 -> 43-48. Chunks are
// balanced (ceil(nz / chunks)) and at most 48 planes (the deferred-node mask
// has 64 bits; longer chunks measured slower).
static int zc_model(int nz, long long tiles, int slots, double k) {
  const double W = (double)tiles * nz / slots;
  const double zs = std::sqrt(k * W);
  int chunks = (int)(nz / std::fmax(zs, 1.0) + 0.5);
  chunks = std::max(chunks, (nz + 47) / 48);
  chunks = std::max(1, std::min(chunks, std::max(1, nz / 4)));
  return (nz + chunks - 1) / chunks;
}

static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
  }
  return sms;
}

int fast_zc(const Geom& g) {
  if (g.dim == 1) return 1;
  if (const char* e = std::getenv("EMRKC_ZC"))  // experiments
    if (*e) return std::max(1, std::min(std::atoi(e), std::min(g.nzl, 48)));
  if (g.dim == 3)  // k_node_tma: 32 x 4 tiles, 5 resident blocks per SM
    return zc_model(g.nzl, ((g.n0 + 31) / 32) * (long long)((g.n1 + 3) / 4), 5 * sm_count(), 7.5);
  const long long tiles = (g.n0 + 127) / 128;
  // 2-D (latency-bound launches): the longest chunk that
  // still gives >= 1.7 waves of resident node blocks
  const long long want = (long long)(1.7 * sm_count() * 5);
  for (int zc = 48; zc >= 4; --zc)
    if (tiles * ((g.nzl + zc - 1) / zc) >= want) return zc > g.nzl ? g.nzl : zc;
  int zc = 16;
  while (zc > 4 && tiles * ((g.nzl + zc - 1) / zc) < 148LL * 5 * 2) zc /= 2;
  return zc > g.nzl ? g.nzl : zc;
}

long long halo_signals_pipe(const Geom& g) {
  if (g.dim == 3) return (long long)((g.n0 + 31) / 32) * ((g.n1 + 3) / 4);
  return (g.n0 + 127) / 128;
}
long long halo_signals_march(const Geom& g) {
  if (g.dim == 3) return (long long)((g.n0 + FBX - 1) / FBX) * ((g.n1 + FBY - 1) / FBY);
  return (g.n0 + FBX - 1) / FBX;
}

namespace {
// Prime level: first / last V plane of y into the neighbours' ghost slots.
// One block per 256 plane points; every block signals the sides it wrote.
__global__ void k_halo_prime(const Geom g, const Halo h, const double* __restrict__ y) {
  const long long i = blockIdx.x * 256LL + threadIdx.x;
  if (i < g.plane) {
    if (h.put_lo) h.put_lo[i] = y[i];
    if (h.put_hi) h.put_hi[i] = y[i + g.plane * (g.nzl - 1)];
  }
  if ((h.put_lo && h.sig_lo) || (h.put_hi && h.sig_hi)) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      if (h.put_lo && h.sig_lo) atomicAdd_system(h.sig_lo, 1ull);
      if (h.put_hi && h.sig_hi) atomicAdd_system(h.sig_hi, 1ull);
    }
  }
}
}  // namespace

long long halo_signals_prime(const Geom& g) { return (g.plane + 255) / 256; }

cudaError_t launch_halo_prime(const Geom& g, const Halo& h, const double* y, cudaStream_t st) {
  k_halo_prime<<<(unsigned)((g.plane + 255) / 256), 256, 0, st>>>(g, h, y);
  return cudaGetLastError();
}

#define FDISPATCH(g, ...)                                   \
  switch ((g).dim) {                                        \
    case 1: { constexpr int D = 1; __VA_ARGS__; break; }    \
    case 2: { constexpr int D = 2; __VA_ARGS__; break; }    \
    default: { constexpr int D = 3; __VA_ARGS__; break; }   \
  }

cudaError_t launch_node_fast(const Geom& g, const Halo& h, const FastArgs& a,
                             bool ion, cudaStream_t st) {
  const dim3 blk(FBX, FBY);
  const bool first = a.j == 1;
  FDISPATCH(g, {
    const dim3 grd = fgrid<D>(g, a.zc);
    if (ion) {
      if (first) k_node_fast<D, 1, 1><<<grd, blk, 0, st>>>(g, h, a);
      else k_node_fast<D, 0, 1><<<grd, blk, 0, st>>>(g, h, a);
    } else {
      if (first) k_node_fast<D, 1, 0><<<grd, blk, 0, st>>>(g, h, a);
      else k_node_fast<D, 0, 0><<<grd, blk, 0, st>>>(g, h, a);
    }
  });
  return cudaGetLastError();
}

// Launch with programmatic stream serialization (PDL) unless EMRKC_PDL=0.
static bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("EMRKC_PDL");
    on = (e && *e) ? (std::atoi(e) != 0) : 1;
  }
  return on != 0;
}

template <typename... P, typename... A>
static cudaError_t launch_k(void (*kern)(P...), dim3 grd, dim3 blk, size_t smem, cudaStream_t st,
                            A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grd;
  cfg.blockDim = blk;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

template <int D, int F, int I>
static cudaError_t launch_pipe_t(const Geom& g, const Halo& h, const FastArgs& a,
                                 cudaStream_t st) {
  using T = PipeTile<D>;
  constexpr size_t smem = pipe_smem_bytes<D, F>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_node_pipe<D, F, I>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  const int chunks = (g.nzl + a.zc - 1) / a.zc;
  const dim3 grd = D == 3 ? dim3((g.n0 + T::TX - 1) / T::TX, (g.n1 + T::TY - 1) / T::TY, chunks)
                          : dim3((g.n0 + T::TX - 1) / T::TX, chunks, 1);
  return launch_k(k_node_pipe<D, F, I>, grd, dim3(T::NT), smem, st, g, h, a);
}

#if EMRKC_EXPERIMENTAL
template <int D, int F, int I>
static cudaError_t launch_persist_t(const Geom& g, const Halo& h, const FastArgs& a,
                                    cudaStream_t st) {
  using T = PipeTile<D>;
  constexpr size_t smem = pipe_smem_bytes<D, F>();
  static int per_sm = 0;
  static int nsm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(k_node_persist<D, F, I>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_node_persist<D, F, I>, T::NT, smem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (per_sm < 1) per_sm = 1;
  }
  const int tiles_x = (g.n0 + T::TX - 1) / T::TX;
  const int tiles_y = D == 3 ? (g.n1 + T::TY - 1) / T::TY : 1;
  const int nchunk = (g.nzl + a.zc - 1) / a.zc;
  const long long items = (long long)tiles_x * tiles_y * nchunk;
  const long long cap = (long long)per_sm * nsm;
  const int grid = (int)(items < cap ? items : cap);
  k_node_persist<D, F, I><<<grid, T::NT, smem, st>>>(g, h, a, (int)items, tiles_x);
  return cudaGetLastError();
}

cudaError_t launch_node_persist(const Geom& g, const Halo& h, const FastArgs& a, bool ion,
                                cudaStream_t st) {
  const bool first = a.j == 1;
  if (g.dim == 3) {
    if (ion) return first ? launch_persist_t<3, 1, 1>(g, h, a, st) : launch_persist_t<3, 0, 1>(g, h, a, st);
    return first ? launch_persist_t<3, 1, 0>(g, h, a, st) : launch_persist_t<3, 0, 0>(g, h, a, st);
  }
  if (g.dim == 2) {
    if (ion) return first ? launch_persist_t<2, 1, 1>(g, h, a, st) : launch_persist_t<2, 0, 1>(g, h, a, st);
    return first ? launch_persist_t<2, 1, 0>(g, h, a, st) : launch_persist_t<2, 0, 0>(g, h, a, st);
  }
  return launch_node_fast(g, h, a, ion, st);
}
#else
// The persistent node kernel is compiled only with -DEMRKC_EXPERIMENTAL=1;
// EMRKC_PIPE=2 selects the TMA / cp.async kernels otherwise (emrkc_capi.cpp).
cudaError_t launch_node_persist(const Geom& g, const Halo& h, const FastArgs& a, bool ion,
                                cudaStream_t st) {
  return launch_node_pipe(g, h, a, ion, st);
}
#endif

template <int D, int F, int I, int AUX>
static cudaError_t launch_node_tma_a(const Geom& g, const Halo& h, const FastArgs& a,
                                     const TmaNode& tm, cudaStream_t st) {
  using T = PipeTile<D>;
  // EMRKC_NODE_PAD: extra dynamic shared memory per block (caps the resident
  // node blocks per SM so that inner-stage blocks of the z-pipelined step
  // fit beside them; experiments only)
  static const size_t pad = [] {
    const char* e = std::getenv("EMRKC_NODE_PAD");
    return e && *e ? (size_t)std::max(0, std::atoi(e)) : (size_t)0;
  }();
  const size_t smem = tma_node_smem_bytes<D, F>(g.naux) + pad;
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(k_node_tma<D, F, I, AUX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = smem;
  }
  const int chunks = (a.z_hi - a.z_lo + a.zc - 1) / a.zc;
  const dim3 grd = D == 3 ? dim3((g.n0 + T::TX - 1) / T::TX, (g.n1 + T::TY - 1) / T::TY, chunks)
                          : dim3((g.n0 + T::TX - 1) / T::TX, chunks, 1);
  return launch_k(k_node_tma<D, F, I, AUX>, grd, dim3(T::NT), smem, st, g, h, a, tm);
}

template <int D, int F, int I>
static cudaError_t launch_node_tma_t(const Geom& g, const Halo& h, const FastArgs& a,
                                     const TmaNode& tm, cudaStream_t st) {
  return g.naux > 0 ? launch_node_tma_a<D, F, I, 1>(g, h, a, tm, st)
                    : launch_node_tma_a<D, F, I, 0>(g, h, a, tm, st);
}

template <int K, int F>
static cudaError_t launch_vin_tb_t(const Geom& g, const Halo& h, const TbArgs& a, const TmaTb& tm,
                                   cudaStream_t st) {
  constexpr size_t smem = tb_smem_bytes<K>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_vin_tb<K, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int chunks = (g.nzl + a.zc - 1) / a.zc;
  const dim3 grd((g.n0 + kTbTX - 1) / kTbTX, (g.n1 + kTbTY - 1) / kTbTY, chunks);
  return launch_k(k_vin_tb<K, F>, grd, dim3(TbTile<K>::NT), smem, st, g, h, a, tm);
}

cudaError_t launch_vin_tb(const Geom& g, const Halo& h, const TbArgs& a, const TmaTb& tm,
                          cudaStream_t st) {
  const bool first = a.j == 1;
  switch (a.m - 1) {
    case 1: return first ? launch_vin_tb_t<1, 1>(g, h, a, tm, st) : launch_vin_tb_t<1, 0>(g, h, a, tm, st);
    case 2: return first ? launch_vin_tb_t<2, 1>(g, h, a, tm, st) : launch_vin_tb_t<2, 0>(g, h, a, tm, st);
    case 3: return first ? launch_vin_tb_t<3, 1>(g, h, a, tm, st) : launch_vin_tb_t<3, 0>(g, h, a, tm, st);
    case 4: return first ? launch_vin_tb_t<4, 1>(g, h, a, tm, st) : launch_vin_tb_t<4, 0>(g, h, a, tm, st);
    default: return cudaErrorInvalidValue;
  }
}

// z-chunk of a k_vin_tb launch: a block marches zc + 2K planes (plus a
// prologue worth ~6) for zc planes of output, and the grid runs in waves of
// (resident blocks per SM) x SMs; pick the chunk count whose waves x march
// length is smallest (chunks of >= 8 planes).
template <int K>
static int tb_slots() {
  static int slots = -1;
  if (slots < 0) {
    int nb = 0, sms = 0, dev = 0;
    cudaFuncSetAttribute(k_vin_tb<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)tb_smem_bytes<K>());
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_vin_tb<K, 1>, TbTile<K>::NT,
                                                      tb_smem_bytes<K>()) != cudaSuccess ||
        cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      nb = 0;
    cudaGetLastError();
    slots = nb > 0 && sms > 0 ? nb * sms : 148 * tb_min_blocks<K>();
  }
  return slots;
}

int tb_zc(const Geom& g, int K) {
  const int slots = K == 1 ? tb_slots<1>() : (K == 2 ? tb_slots<2>() : (K == 3 ? tb_slots<3>() : tb_slots<4>()));
  const long long tiles = halo_signals_tb(g);
  const int nz = g.nzl;
  int best_zc = nz;
  long long best = -1;
  for (int chunks = 1; chunks <= nz; ++chunks) {
    const int zc = (nz + chunks - 1) / chunks;
    if (zc < 8 && chunks > 1) break;
    const int real = (nz + zc - 1) / zc;
    const long long waves = (tiles * real + slots - 1) / slots;
    const long long cost = waves * (zc + 2 * K + 6);
    if (best < 0 || cost < best) {
      best = cost;
      best_zc = zc;
    }
  }
  return best_zc;
}

long long halo_signals_tb(const Geom& g) {
  return (long long)((g.n0 + kTbTX - 1) / kTbTX) * ((g.n1 + kTbTY - 1) / kTbTY);
}

cudaError_t launch_node_tma(const Geom& g, const Halo& h, const FastArgs& a, const TmaNode& tm,
                            bool ion, cudaStream_t st) {
  const bool first = a.j == 1;
  if (g.dim == 3) {
    if (ion) return first ? launch_node_tma_t<3, 1, 1>(g, h, a, tm, st) : launch_node_tma_t<3, 0, 1>(g, h, a, tm, st);
    return first ? launch_node_tma_t<3, 1, 0>(g, h, a, tm, st) : launch_node_tma_t<3, 0, 0>(g, h, a, tm, st);
  }
  if (ion) return first ? launch_node_tma_t<2, 1, 1>(g, h, a, tm, st) : launch_node_tma_t<2, 0, 1>(g, h, a, tm, st);
  return first ? launch_node_tma_t<2, 1, 0>(g, h, a, tm, st) : launch_node_tma_t<2, 0, 0>(g, h, a, tm, st);
}

// k_node_pair (3-D, whole grid, HH proper): z-chunk for 64 x 4 tiles at 4
// (FIRST) / 2 resident blocks per SM, same 1.7-wave floor as fast_zc.
// Tile width of k_node_pair on this grid: 32 x 8 tiles when they waste at
// least 5% fewer lanes than 64 x 4 tiles (EMRKC_PAIR_TX: 32 / 64, experiments).
int pair_tx(const Geom& g) {
  if (const char* e = std::getenv("EMRKC_PAIR_TX"))
    if (*e) return std::atoi(e) == 32 ? 32 : 64;
  const double c64 = (double)((g.n0 + 63) / 64 * 64) * ((g.n1 + 3) / 4 * 4);
  const double c32 = (double)((g.n0 + 31) / 32 * 32) * ((g.n1 + 7) / 8 * 8);
  return c32 * 1.05 <= c64 ? 32 : 64;
}

int pair_zc(const Geom& g, bool first, bool force) {
  if (const char* e = std::getenv("EMRKC_PAIR_ZC"))  // experiments
    if (*e) return std::max(1, std::min(std::atoi(e), std::min(g.nzl, kMaxZc)));
  const int tx = pair_tx(g), ty = kPairNT * 2 / tx;
  const long long tiles = (long long)((g.n0 + tx - 1) / tx) * ((g.n1 + ty - 1) / ty);
  const int slots = sm_count() * (first ? 4 : 2);
  // fewer blocks than one wave of slots: k_node_tma's smaller tiles fill the GPU better
  if (!force && tiles * ((g.nzl + 3) / 4) < slots) return 0;
  // small grids (< 12 planes per slot): the shortest chunks (sweep N = 100:
  // zc 4 / 7 / 10 -> 30.0 / 33.4 / 36.4 us per launch)
  if ((double)tiles * g.nzl / slots < 12.0) return std::min(g.nzl, 4);
  return zc_model(g.nzl, tiles, slots, 3.75);
}

template <int F, int I, int TXW>
static cudaError_t launch_node_pair_t(const Geom& g, const Halo& h, const FastArgs& a,
                                      const TmaNode& tm, cudaStream_t st) {
  using P = PairTile<TXW>;
  constexpr size_t smem = pair_smem_bytes<F, TXW>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_node_pair<F, I, TXW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  const int chunks = (a.z_hi - a.z_lo + a.zc - 1) / a.zc;
  const dim3 grd((g.n0 + P::TX - 1) / P::TX, (g.n1 + P::TY - 1) / P::TY, chunks);
  return launch_k(k_node_pair<F, I, TXW>, grd, dim3(kPairNT), smem, st, g, h, a, tm);
}

template <int TXW>
static cudaError_t launch_node_pair_w(const Geom& g, const Halo& h, const FastArgs& a,
                                      const TmaNode& tm, bool ion, cudaStream_t st) {
  const bool first = a.j == 1;
  if (ion)
    return first ? launch_node_pair_t<1, 1, TXW>(g, h, a, tm, st)
                 : launch_node_pair_t<0, 1, TXW>(g, h, a, tm, st);
  return first ? launch_node_pair_t<1, 0, TXW>(g, h, a, tm, st)
               : launch_node_pair_t<0, 0, TXW>(g, h, a, tm, st);
}

cudaError_t launch_node_pair(const Geom& g, const Halo& h, const FastArgs& a, const TmaNode& tm,
                             bool ion, cudaStream_t st) {
  return pair_tx(g) == 32 ? launch_node_pair_w<32>(g, h, a, tm, ion, st)
                          : launch_node_pair_w<64>(g, h, a, tm, ion, st);
}

cudaError_t launch_step_x(const Geom& g, const XArgs& a, const TmaX& tm, cudaStream_t st) {
  constexpr size_t smem = xstep_smem_bytes();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_step_x, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int chunks = (g.nzl + a.f.zc - 1) / a.f.zc;
  const dim3 grd((g.n0 + kPairTX - 1) / kPairTX, (g.n1 + kPairTY - 1) / kPairTY, chunks);
  return launch_k(k_step_x, grd, dim3(kPairNT), smem, st, g, a, tm);
}

template <int D, int L, int F>
static cudaError_t launch_vin_tma_t(const Geom& g, const Halo& h, const FastInnerArgs& a,
                                    const TmaVin& tm, cudaStream_t st) {
  using T = PipeTile<D>;
  constexpr size_t smem = tma_vin_smem_bytes<D>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_vin_tma<D, L, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  const int chunks = (a.z_hi - a.z_lo + a.zc - 1) / a.zc;
  const dim3 grd = D == 3 ? dim3((g.n0 + T::TX - 1) / T::TX, (g.n1 + T::TY - 1) / T::TY, chunks)
                          : dim3((g.n0 + T::TX - 1) / T::TX, chunks, 1);
  return launch_k(k_vin_tma<D, L, F>, grd, dim3(T::NT), smem, st, g, h, a, tm);
}

template <int L, int F, int R>
static cudaError_t launch_vin_tma_r_t(const Geom& g, const Halo& h, const FastInnerArgs& a,
                                      const TmaVin& tm, cudaStream_t st) {
  using T = VinTileR<R>;
  const int nb = (a.um1 == a.d1 ? 0 : 1) + (a.um2 ? 1 : 0) + (L ? (F ? 1 : 2) : 0);
  const size_t smem = tma_vin_r_smem_bytes<R>(nb);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_vin_tma_r<L, F, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)tma_vin_r_smem_bytes<R>(4));
    attr = true;
  }
  const int chunks = (a.z_hi - a.z_lo + a.zc - 1) / a.zc;
  const dim3 grd((g.n0 + T::TX - 1) / T::TX, (g.n1 + T::TY - 1) / T::TY, chunks);
  return launch_k(k_vin_tma_r<L, F, R>, grd, dim3(T::NT), smem, st, g, h, a, tm);
}

int vin_rows(const Geom& g) { return g.dim == 3 ? EMRKC_VIN_R : 1; }
long long halo_signals_vin(const Geom& g) {
  if (g.dim != 3) return halo_signals_pipe(g);
  const int ty = 4 * EMRKC_VIN_R;
  return (long long)((g.n0 + 31) / 32) * ((g.n1 + ty - 1) / ty);
}

cudaError_t launch_vin_tma(const Geom& g, const Halo& h, const FastInnerArgs& a, const TmaVin& tm,
                           cudaStream_t st) {
  const bool last = a.k == a.m, first = a.j == 1;
  if (g.dim == 3 && EMRKC_VIN_R > 1) {
    constexpr int R = EMRKC_VIN_R > 1 ? EMRKC_VIN_R : 2;
    if (!last) return launch_vin_tma_r_t<0, 0, R>(g, h, a, tm, st);
    return first ? launch_vin_tma_r_t<1, 1, R>(g, h, a, tm, st)
                 : launch_vin_tma_r_t<1, 0, R>(g, h, a, tm, st);
  }
#if EMRKC_VIN_R <= 1  // 3-D one row per thread: measured slower than k_vin_tma_r
  if (g.dim == 3) {
    if (!last) return launch_vin_tma_t<3, 0, 0>(g, h, a, tm, st);
    return first ? launch_vin_tma_t<3, 1, 1>(g, h, a, tm, st) : launch_vin_tma_t<3, 1, 0>(g, h, a, tm, st);
  }
#endif
  if (!last) return launch_vin_tma_t<2, 0, 0>(g, h, a, tm, st);
  return first ? launch_vin_tma_t<2, 1, 1>(g, h, a, tm, st) : launch_vin_tma_t<2, 1, 0>(g, h, a, tm, st);
}

cudaError_t launch_node_pipe(const Geom& g, const Halo& h, const FastArgs& a, bool ion,
                             cudaStream_t st) {
  const bool first = a.j == 1;
  if (g.dim == 3) {
    if (ion) return first ? launch_pipe_t<3, 1, 1>(g, h, a, st) : launch_pipe_t<3, 0, 1>(g, h, a, st);
    return first ? launch_pipe_t<3, 1, 0>(g, h, a, st) : launch_pipe_t<3, 0, 0>(g, h, a, st);
  }
  if (g.dim == 2) {
    if (ion) return first ? launch_pipe_t<2, 1, 1>(g, h, a, st) : launch_pipe_t<2, 0, 1>(g, h, a, st);
    return first ? launch_pipe_t<2, 1, 0>(g, h, a, st) : launch_pipe_t<2, 0, 0>(g, h, a, st);
  }
  return launch_node_fast(g, h, a, ion, st);
}

template <int D, int L, int F>
static cudaError_t launch_vin_pipe_t(const Geom& g, const Halo& h, const FastInnerArgs& a,
                                     cudaStream_t st) {
  using T = PipeTile<D>;
  constexpr size_t smem = vin_smem_bytes<D>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_vin_pipe<D, L, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  const int chunks = (g.nzl + a.zc - 1) / a.zc;
  const dim3 grd = D == 3 ? dim3((g.n0 + T::TX - 1) / T::TX, (g.n1 + T::TY - 1) / T::TY, chunks)
                          : dim3((g.n0 + T::TX - 1) / T::TX, chunks, 1);
  return launch_k(k_vin_pipe<D, L, F>, grd, dim3(T::NT), smem, st, g, h, a);
}

cudaError_t launch_vin_pipe(const Geom& g, const Halo& h, const FastInnerArgs& a,
                            cudaStream_t st) {
  const bool last = a.k == a.m, first = a.j == 1;
  if (g.dim == 3) {
    if (!last) return launch_vin_pipe_t<3, 0, 0>(g, h, a, st);
    return first ? launch_vin_pipe_t<3, 1, 1>(g, h, a, st) : launch_vin_pipe_t<3, 1, 0>(g, h, a, st);
  }
  if (g.dim == 2) {
    if (!last) return launch_vin_pipe_t<2, 0, 0>(g, h, a, st);
    return first ? launch_vin_pipe_t<2, 1, 1>(g, h, a, st) : launch_vin_pipe_t<2, 1, 0>(g, h, a, st);
  }
  return launch_vin_fast(g, h, a, st);
}

cudaError_t launch_vin_fast(const Geom& g, const Halo& h, const FastInnerArgs& a,
                            cudaStream_t st) {
  const dim3 blk(FBX, FBY);
  const bool last = a.k == a.m;
  const bool first = a.j == 1;
  FDISPATCH(g, {
    const dim3 grd = fgrid<D>(g, a.zc);
    if (!last) k_vin_fast<D, 0, 0><<<grd, blk, 0, st>>>(g, h, a);
    else if (first) k_vin_fast<D, 1, 1><<<grd, blk, 0, st>>>(g, h, a);
    else k_vin_fast<D, 1, 0><<<grd, blk, 0, st>>>(g, h, a);
  });
  return cudaGetLastError();
}


#if EMRKC_EXPERIMENTAL
// Fused s = 1, m = 2 step: resident blocks per SM of k_fused2 (0 if it
// cannot run) and the cooperative launch.
int fused_blocks_per_sm() {
  static int nb = -1;
  if (nb < 0) {
    cudaFuncSetAttribute(k_fused2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)fused_smem_bytes());
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fused2, kFuNT,
                                                      fused_smem_bytes()) != cudaSuccess)
      nb = 0;
    cudaGetLastError();
  }
  return nb;
}

cudaError_t launch_fused2(const Geom& g, const FusedArgs& a, const TmaFused& tm, cudaStream_t st) {
  if (fused_blocks_per_sm() < 1) return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.ntx * a.nty * a.nzc));
  cfg.blockDim = dim3(kFuNT);
  cfg.dynamicSmemBytes = fused_smem_bytes();
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // co-residency or an error, never a hang
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_fused2, g, a, tm);
}

#else
// k_fused2 is compiled only with -DEMRKC_EXPERIMENTAL=1 (EMRKC_FUSED=1 then
// keeps the two-kernel step).
int fused_blocks_per_sm() { return 0; }
cudaError_t launch_fused2(const Geom&, const FusedArgs&, const TmaFused&, cudaStream_t) {
  return cudaErrorNotSupported;
}
#endif

}  // namespace emrkc_k
