// kernels.h — host-side launch interface of the emRKC sm_100a kernels.
// Internal to libemrkc_b200.so (not part of the C ABI).
#pragma once

#include <cmath>

#include <cstdint>

#include <cuda.h>
#include <cuda_runtime.h>

namespace emrkc_k {

constexpr unsigned long long kNoEvent = ~0ull;
// Lowest abort ordinal a launch of outer stage j can raise when its first
// inner stage is k0 (ordinal = code_base + (j-1)(m+1) + k; the outer check
// is k = m+1, the step's norm guard s(m+1)+1). A launch skips its work only
// on an event BELOW this floor, i.e. from an earlier level (an earlier step,
// or an earlier stage of this step). Events at or above it come from other
// blocks / z-chunks of the same level or from this step's guard, and must
// not stop the remaining blocks: the first failing check in program order
// and the guard step's full state depend on every block finishing.
__host__ __device__ __forceinline__ unsigned long long level_floor(
    unsigned long long code_base, int j, int m, int k0) {
  return code_base + (unsigned long long)((j - 1) * (m + 1) + k0);
}
constexpr int kMaxStages = 512;  // per rkc iteration (coefficients in params)

// Geometry of the local z-slab (the whole grid when not partitioned).
// The slab axis is axis dim-1; unused axes have extent 1.
struct Geom {
  int dim;
  int n0, n1, n2;         // local extents per axis (slab axis local count)
  int nzl, nzg, zoff;     // slab axis: local count, global count, offset
  long long plane;        // stride of the slab axis
  long long nn;           // local nodes
  double w[3];            // sigma_a / (chi C_m dx_a^2)
  double wc;              // -2 sum_a w_a (fast kernels)
  double inv_Cm, Cm;
  int st_lo[3], st_hi[3]; // stimulus node box per axis (global, inclusive)
  int naux;               // auxiliary fields (EMRKC_MODEL_HH_AUX; 0 for HH)
  int nf;                 // SoA fields of the state: 4 + naux
};

// Ghost planes of the V field consumed by one stencil level.
struct Halo {
  const double* lo;   // plane z = zoff-1 (null: global boundary)
  const double* hi;   // plane z = zoff+nzl
  double* put_lo;     // where my first plane goes (lower neighbour's hi ghost)
  double* put_hi;     // where my last plane goes (upper neighbour's lo ghost)
  // Cross-process protocol (null in-process, where stream order suffices):
  // a block that put a plane bumps the neighbour's arrival counter after a
  // system-scope fence; a block that reads a ghost plane first waits until
  // its own counter reaches `expect_*`.
  unsigned long long* sig_lo;        // lower neighbour's counter for its hi ghost
  unsigned long long* sig_hi;        // upper neighbour's counter for its lo ghost
  const unsigned long long* wait_lo; // my counter for my lo ghost
  const unsigned long long* wait_hi;
  unsigned long long expect_lo, expect_hi;
  unsigned long long* timeout_flag;  // the abort word (code 0 = wait timed out)
  // Wide d_1 halo of the temporally blocked inner stages on slabs (north_star
  // (4): K-plane halos when K stages are blocked). kput > 0: the inner-stage-1
  // node kernel stores its first / last kput planes of d_1 into the
  // neighbours' d_1 ghosts instead of one plane into put_lo / put_hi:
  // plane z < kput to kput_lo + z * plane (the lower neighbour's upper ghost),
  // plane z >= nzl - kput to kput_hi + (z - nzl + kput) * plane. A block
  // signals one arrival per plane it stored, so a side expects
  // kput * halo_signals_pipe arrivals whatever the sender's z-chunking.
  double* kput_lo;
  double* kput_hi;
  int kput;
};

// One outer stage of emRKC: pointers and coefficients.
struct StageArgs {
  const double* g1;   // g_{j-1} (state layout, 4 blocks)
  const double* g2;   // g_{j-2} (null for j == 1)
  double* out;        // g_j
  double* fs;         // m >= 2: frozen slow V term (n)
  double* ye;         // m >= 2: y_E gate blocks (3n)
  double* u[3];       // m >= 2: inner V stages (rotating)
  double eta, inv_eta;
  double stim;        // stimulus rate at this stage's time (0 if inactive)
  double mudt, nu, kappa;  // outer: mu_j*dt, nu_j, kappa_j
  int j, s, m;
  // inner coefficients (index 1..m): mu'_k*eta, nu'_k, kappa'_k
  const double* in_mueta;
  const double* in_nu;
  const double* in_kappa;
  unsigned long long code_base;  // step_in_run * stride
  unsigned long long* event;     // first abort/guard event (atomicMin)
  unsigned long long* gate_slot; // [2]: ordered min, max for this step
  const unsigned long long* gate_prev;  // range slot of everything before this step (or null)
  int last;                      // j == s: guard + gate range
};

// mRKC (P/src/multirate.cpp:60-76,158-171) with the stiff-gate split of
// run_simulation (P/src/simulate.cpp:132-150): inner stage k of outer j.
struct MrkcArgs {
  const double* g1;   // g_{j-1} = u_0 (state layout)
  const double* g2;   // g_{j-2} (j >= 2)
  double* out;        // g_j (written at k == m)
  double* fs;         // frozen slow term f_S_with_gates(g_{j-1}) (4 blocks)
  const double* um1;  // u_{k-1} (4 blocks; g_{j-1} for k == 1)
  const double* um2;  // u_{k-2} (k >= 2; g_{j-1} for k == 2)
  double* uk;         // u_k (k < m)
  double eta, mueta, nu, kappa;  // inner: eta, mu'_k eta, nu'_k, kappa'_k
  double mudt, onu, okappa;      // outer: mu_j dt, nu_j, kappa_j
  double stim;                   // stimulus rate at the outer stage time
  int stiff;                     // gate mask of the fast part
  int j, k, m, s, last;
  unsigned long long code_base;
  unsigned long long* event;
};
cudaError_t launch_mrkc_stage(const Geom& g, const MrkcArgs& a, cudaStream_t st);

// IMEX-RL (P/src/baselines.cpp:132-190): Rush-Larsen gates, then
// (I - dt D) V_new = V + dt v_rhs by Jacobi-preconditioned CG in
// sqrt(w)-scaled coordinates (w: trapezoid node weights). Device scalars:
struct CgScalars {
  double nb2;      // ||b||^2
  double rz, pq, rr;
  double alpha, beta;
  double tol;      // rel_tol ||b||
  long long it, max_it;
  int done, converged;
};
// vectors (n_nodes each): b, x, r, z, p, q
cudaError_t launch_imex_prep(const Geom& g, const double* y, double dt, double stim,
                             double* out, double* b, double* x, double* partial, int nblocks,
                             cudaStream_t st);
cudaError_t launch_cg_init(const Geom& g, double dt, double diag, const double* b,
                           const double* x, double* r, double* z, double* p, double* partial,
                           int nblocks, CgScalars* cs, double rel_tol, long long max_it,
                           const double* partial_b, cudaStream_t st);
cudaError_t launch_cg_iter(const Geom& g, double dt, double diag, double* x, double* r,
                           double* z, double* p, double* q, double* partial, int nblocks,
                           CgScalars* cs, cudaStream_t st);
cudaError_t launch_cg_finish(const Geom& g, const double* x, double* out, const CgScalars* cs,
                             cudaStream_t st);
cudaError_t launch_v_guard(long long nn, const double* y, int* flag, cudaStream_t st);
// diffusion_apply of the unit vector at node 0, component 0 (the constant
// diagonal of the reflection stencil, baselines.cpp:171-177)
double diffusion_diag(const Geom& g);

// Arguments of the fast kernels (kernels_fast.cu): one outer stage j.
struct FastArgs {
  const double* g1;   // g_{j-1}
  const double* g2;   // g_{j-2} (j >= 2)
  double* out;        // g_j (m == 1: all blocks; m >= 2: gate blocks)
  double* fs;         // unused (kept for layout stability)
  double* u1;         // m >= 2: d_1 = u_1 - V (increment form, see FastInnerArgs)
  double eta;
  double stim;        // stimulus rate at the stage time (0 if inactive)
  double cG;          // mu_j dt / eta   (gate rows: g_j = base + cG (y_E - z))
  double cV;          // cG * mu'_1 eta  (m == 1: V of g_j = base + cV (f_F + f_S))
  double mue1;        // mu'_1 eta       (m >= 2: u_1 = V + mue1 (f_F + f_S))
  double nu, kappa;   // outer nu_j, kappa_j (j >= 2)
  double cA;          // aux rows: mu_j dt c_m (g_j = base + cA g_S; inner c_m)
  double vmid, vfast; // fast ionic path iff |V - vmid| <= vfast (fast_window)
  int j, m, s, last, zc;
  int exex;           // EXEX-RL step: non-finite values are not aborts (guard only)
  int z_lo, z_hi;     // k_node_tma: local planes [z_lo, z_hi) of this launch (0, nzl: all)
  unsigned long long code_base;
  unsigned long long* event;
  unsigned long long* gate_slot;
  // k_node_pair: the gate-range slot that holds the range of everything
  // before this step of the run (initial state and earlier steps), or null.
  // With it the kernel's slot becomes cumulative (prev folded in) and values
  // whose high words lie strictly inside prev's skip the FP64 min / max.
  const unsigned long long* gate_prev;
  // k_node_pair: integer-pipe form of the window test on V's high word hi:
  // (int)hi < vq_pos && (unsigned)hi < vq_neg implies vlo < V < vhi. Nodes
  // that fail it (including the few inside the window but past the high-word
  // bounds) take the per-node path, which applies the exact test.
  int vq_pos;
  unsigned vq_neg;
};

// Whole-run resident kernel for small grids (s = m = 1; emRKC standard /
// progressive, EXEX-RL): one cooperative launch runs all steps of an
// emrkc_run. Every thread keeps its nodes' gates in registers, V ping-pongs
// through two L2-resident fields, and a grid barrier separates the steps;
// the node arithmetic is k_node_tma's, operation for operation.
struct ResidentArgs {
  FastArgs f;                    // stage coefficients (g1/g2/out/stim unused)
  const double* y_in;            // state at the run start (4 blocks)
  double* y_out;                 // state the run ends on (4 blocks)
  double* vbuf;                  // [2][nn] V ping-pong
  const double* stim;            // stimulus rate per step [nsteps]
  long long nsteps;
  unsigned long long stride;     // abort-ordinal stride per step
  unsigned long long* slots;     // gate range of the accepted steps -> slots[0..1]
  unsigned* bar;                 // [2] grid-barrier arrival counters (zeroed by the host)
};
// Largest grid the resident kernel takes on this device (0: none).
long long resident_capacity(int dim);
cudaError_t launch_resident(const Geom& g, const ResidentArgs& a, cudaStream_t st);

// Inner stages in increment form: d_k = u_k - V (V = y_E's V block), so
// d_k = nu' d_{k-1} + kappa' d_{k-2} + mu'_k eta (a + f_F(d_{k-1})) with
// a = (f_F + f_S)(y_E) = d_1 / (mu'_1 eta) and d_0 = 0 (f_F is linear and
// nu' + kappa' = 1). Stage 1 stores only d_1; no fs field is needed.
struct FastInnerArgs {
  const double* um1;  // d_{k-1} (stencil field)
  const double* um2;  // d_{k-2} (null when k == 2: d_0 = 0)
  const double* d1;   // d_1 (gives a)
  double inv_mue1;    // 1 / (mu'_1 eta)
  double* uk;         // k < m: d_k
  const double* g1v;  // k == m: V of g_{j-1}, g_{j-2}
  const double* g2v;
  double* outv;       // k == m: V block of g_j
  double mueta, nu, kappa;  // inner mu'_k eta, nu'_k, kappa'_k
  double onu, okappa, cG;   // outer nu_j, kappa_j, mu_j dt / eta
  int j, k, m, s, last, zc;
  int z_lo, z_hi;     // k_vin_tma*: local planes [z_lo, z_hi) of this launch
  unsigned long long code_base;
  unsigned long long* event;
};

// Fused s = 1, m = 2 step (k_fused2, kernels_fast.cu): node update + inner
// stage 2 + outer update in one pass; persistent co-resident grid of
// ntx x nty column tiles (kFuTX wide, <= kFuTY rows) x nzc z-chunks, d_1
// tile edges exchanged through an L2-resident ring with per-block flags.
constexpr int kFuTX = 64, kFuTY = 14, kFuNT = 256;
struct FusedArgs {
  FastArgs f;                 // node phase (j = 1, ION): g1, out, eta, stim, cG, mue1, window, events
  double inv_mue1;            // 1 / (mu'_1 eta)
  double mueta2, nu2;         // inner stage 2: mu'_2 eta, nu'_2
  double cG2;                 // outer: mu_1 dt / eta
  double* xch;                // exchange ring [blocks][4 planes][4 sides][kFuTX]
  unsigned long long* flags;  // [blocks]: epoch + (last published plane + 1)
  unsigned long long epoch;   // strictly increasing per launch (flags never reset)
  int ntx, nty, nzc;
};
struct TmaFused {
  CUtensorMap v;      // V of g_0, box (kFuTX + 4, kFuTY + 2, 1)
  CUtensorMap gates;  // all fields of g_0, box (kFuTX, kFuTY, 1, 3) from field 1
};
int fused_blocks_per_sm();
cudaError_t launch_fused2(const Geom& g, const FusedArgs& a, const TmaFused& tm, cudaStream_t st);

// Temporally blocked inner stages: one pass runs stages k = 2..m (m - 1 = K
// fused V-only stages, 2 <= K <= kTbMaxK) of outer stage j (3-D, whole-grid
// handles). Stage k is computed on the tile plus a halo of K + 1 - k cells
// (recomputed), so only d_1 (halo K), V of g_{j-1} / g_{j-2} and V of g_j
// touch HBM.
constexpr int kTbMaxK = 4, kTbTX = 32, kTbTY = 16;
constexpr int tb_hx(int K) { return (K + 1) & ~1; }  // x halo of the d_1 box: K rounded up to even
struct TbArgs {
  double mueta[kTbMaxK + 2], nu[kTbMaxK + 2], kappa[kTbMaxK + 2];  // mu'_k eta, nu'_k, kappa'_k (k = 0..m)
  const double* g1v;   // V block of g_{j-1}
  const double* g2v;   // V block of g_{j-2} (j >= 2)
  double* outv;        // V block of g_j
  double inv_mue1;     // 1 / (mu'_1 eta)
  double onu, okappa, cG;  // outer nu_j, kappa_j, mu_j dt / eta
  int j, m, s, last, zc;
  unsigned long long code_base;
  unsigned long long* event;
};
struct TmaTb {
  CUtensorMap d1;      // d_1, box (kTbTX + 2 tb_hx(K), kTbTY + 2K, 1)
  CUtensorMap d1lo;    // slabs: K ghost planes of d_1 below (global z0 - K ..), box as d1
  CUtensorMap d1hi;    // K ghost planes above (global z1 ..)
};
// Slabs (h.lo / h.hi non-null: the d_1 ghosts of that face, K planes each):
// the march extends K planes into the ghosts instead of mirroring, and the
// final stage stores its boundary V planes into put_lo / put_hi (one arrival
// per block and side, halo_signals_tb).
cudaError_t launch_vin_tb(const Geom& g, const Halo& h, const TbArgs& a, const TmaTb& tm,
                          cudaStream_t st);
long long halo_signals_tb(const Geom& g);
int tb_zc(const Geom& g, int K);  // wave-aware z-chunk of a k_vin_tb launch

// TMA descriptors of one k_node_tma launch (host-encoded, passed as a
// __grid_constant__ parameter). Boxes: V tile + 1-cell halo, gate fields,
// g_{j-2} fields, ghost planes.
struct TmaNode {
  CUtensorMap v;       // V block of g_{j-1}, box (TX+4, TY+2, 1)
  CUtensorMap gates;   // all fields of g_{j-1}, box (TX, TY, 1, 3) from field 1
  CUtensorMap g2;      // all fields of g_{j-2}, box (TX, TY, 1, 4)
  CUtensorMap glo;     // ghost plane below, box (TX+4, TY+2)
  CUtensorMap ghi;     // ghost plane above
};
struct TmaVin {
  CUtensorMap u;       // d_{k-1}, box (TX+4, TY+2, 1)
  CUtensorMap d1;      // center boxes (TX, TY, 1)
  CUtensorMap um2;
  CUtensorMap g1v;
  CUtensorMap g2v;
  CUtensorMap glo, ghi;
};
// Tile shape of the staged kernels (x, y per block; 2-D grids use TX2 x 1).
constexpr int kTX3 = 32, kTY3 = 4, kTX2 = 128;

// z-chunk length of the staged kernels: k_node_tma's deferred-node mask is
// 64 bits wide; k_node_pipe / k_node_persist keep a 32-bit one (kMaxZcPipe).
constexpr int kMaxZc = 64;
constexpr int kMaxZcPipe = 32;

// Window of V where the fast ionic path (fast_math.cuh, hh_expeuler_fast)
// is valid for this eta: eta * (alpha + beta) <= 600 for every gate and every
// exponential argument within +-700 (derivation in fast_math.cuh). The lower
// end is solved on the host from the full rate sums (emrkc_capi.cpp
// fast_window); the upper end is closed-form:
inline double fast_vhi(double eta) { return std::fmin(10000.0, 6000.0 / eta - 80.0); }
int fast_zc(const Geom& g);
// Signals per level that a neighbour receives from one launch of each kernel
// family (blocks that hold the boundary plane of their slab).
long long halo_signals_pipe(const Geom& g);
long long halo_signals_march(const Geom& g);
long long halo_signals_prime(const Geom& g);
// Copies the first / last V plane of `y` into the neighbours' ghost slots
// and signals (prime level of a distributed run).
cudaError_t launch_halo_prime(const Geom& g, const Halo& h, const double* y,
                              cudaStream_t st);
cudaError_t launch_node_fast(const Geom& g, const Halo& h, const FastArgs& a,
                             bool ion, cudaStream_t st);
cudaError_t launch_node_pipe(const Geom& g, const Halo& h, const FastArgs& a,
                             bool ion, cudaStream_t st);
cudaError_t launch_node_persist(const Geom& g, const Halo& h, const FastArgs& a,
                                bool ion, cudaStream_t st);
cudaError_t launch_node_tma(const Geom& g, const Halo& h, const FastArgs& a,
                            const TmaNode& tm, bool ion, cudaStream_t st);
// Pair-per-thread node kernel (3-D whole grids, HH proper): TMA boxes of
// 64 x 4 tiles (tm.v: (68, 6, 1), tm.gates: (64, 4, 1, 3), tm.g2: (64, 4, 1,
// 4), ghost planes (68, 6)). pair_zc: its z-chunk, 0 if the grid gives too few
// blocks (the caller keeps k_node_tma) unless forced (tests).
constexpr int kPairXMul = 2;  // k_step_x: tile width in units of kTX3
int pair_tx(const Geom& g);    // k_node_pair tile width on this grid: 64 (x 4 rows) or 32 (x 8 rows)
int pair_zc(const Geom& g, bool first, bool force);
cudaError_t launch_node_pair(const Geom& g, const Halo& h, const FastArgs& a, const TmaNode& tm,
                             bool ion, cudaStream_t st);
// Cross-step fusion of the s = 1, m = 2 step (k_step_x, EMRKC_XSTEP=1): inner
// stage 2 of step n and the node update of step n + 1 in one launch.
struct XArgs {
  FastArgs f;           // update of step n + 1 (j = 1, ION): g1 = y_{n+1}'s buffer (its gate
                        // fields are final), out = y_{n+2}'s buffer, u1 = d_1 of step n + 1
  const double* vn;     // V of y_n
  const double* d1;     // d_1 of step n
  double* vout;         // V of y_{n+1} (field 0 of f.g1's buffer)
  double inv_mue1, mueta2, nu2, cG2;  // 1/(mu'_1 eta), mu'_2 eta, nu'_2, mu_1 dt / eta
  unsigned long long code_prev;       // abort-code base of step n
};
struct TmaX {
  CUtensorMap d1;     // d_1 of step n, box (68, 8, 1) at (x0 - 2, y0 - 2)
  CUtensorMap gates;  // fields of y_{n+1}'s buffer, box (64, 4, 1, 3) from field 1
};
cudaError_t launch_step_x(const Geom& g, const XArgs& a, const TmaX& tm, cudaStream_t st);
// Rows per thread of the 3-D inner-stage kernel (its TMA boxes are
// (TX+4) x (4 rows + 2) and TX x 4 rows, rows = vin_rows); 1 in 2-D.
int vin_rows(const Geom& g);
long long halo_signals_vin(const Geom& g);  // arrivals per side of a launch_vin_tma level
cudaError_t launch_vin_tma(const Geom& g, const Halo& h, const FastInnerArgs& a,
                           const TmaVin& tm, cudaStream_t st);
cudaError_t launch_vin_fast(const Geom& g, const Halo& h,
                            const FastInnerArgs& a, cudaStream_t st);
cudaError_t launch_vin_pipe(const Geom& g, const Halo& h,
                            const FastInnerArgs& a, cudaStream_t st);

// Launch helpers (all asynchronous on `st`). fast: shared-transcendental
// ionic evaluation (hh_fast) instead of the reference-order one.
cudaError_t launch_stage_m1(const Geom& g, const Halo& h, const StageArgs& a,
                            int fast, cudaStream_t st);
cudaError_t launch_stage_first(const Geom& g, const Halo& h,
                               const StageArgs& a, int fast, cudaStream_t st);
cudaError_t launch_stage_inner(const Geom& g, const Halo& h,
                               const StageArgs& a, int k, int fast,
                               cudaStream_t st);

// Operator evaluations on the device (for parity / power iteration).
cudaError_t launch_rhs(const Geom& g, const Halo& h, int which,
                       const double* y, double stim, double* out,
                       cudaStream_t st);
cudaError_t launch_exp_part(const Geom& g, const double* y, double* lam,
                            double* yinf, cudaStream_t st);

// Power-iteration step: vout = f(y + q v) - fy, partial sums of vout^2.
// ghost_y / ghost_v: slab-axis ghost planes of y_V and v_V (nullable).
cudaError_t launch_power(const Geom& g, int which, const double* y,
                         const double* v, double q,
                         const double* fy, double stim, double* vout,
                         const double* gy_lo, const double* gy_hi,
                         const double* gv_lo, const double* gv_hi,
                         double* partial, int nblocks, cudaStream_t st);
// Trapezoid-weighted sum((a - b)^2), sum(b^2) of one node field -> out2[0..1]
// (partial: 2 * nblocks doubles).
cudaError_t launch_rel_l2(const Geom& g, const double* a, const double* b, double* partial,
                          int nblocks, double* out2, cudaStream_t st);
cudaError_t launch_norm2_partial(const double* x, long long len,
                                 double* partial, int nblocks,
                                 cudaStream_t st);
cudaError_t launch_sum_partials(const double* partial, int nblocks,
                                double* out, cudaStream_t st);
// Serial-order sum of squares (the reference's norm2 order), continuing
// from acc, result to *out (device).
cudaError_t launch_sumsq_serial(const double* x, long long len, double acc, double* out,
                                cudaStream_t st);

// Gate range of a state (ordered-u64 min/max into slot[0..1]) and
// max |V| (ordered) into *vmax (nullable).
cudaError_t launch_gate_range(const Geom& g, const double* y,
                              unsigned long long* slot, cudaStream_t st);
cudaError_t launch_fold_events(unsigned long long* dst,
                               unsigned long long* const* src, int n,
                               cudaStream_t st);
cudaError_t launch_fill_u64(unsigned long long* p, long long n,
                            unsigned long long v, cudaStream_t st);

int power_blocks();  // fixed grid of the deterministic reductions

// Ordered-u64 encoding of doubles for atomic min/max.
__host__ __device__ inline unsigned long long ord_of(double x) {
  unsigned long long b;
#ifdef __CUDA_ARCH__
  b = (unsigned long long)__double_as_longlong(x);
#else
  __builtin_memcpy(&b, &x, 8);
#endif
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double double_of(unsigned long long o) {
  unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  double x;
#ifdef __CUDA_ARCH__
  x = __longlong_as_double((long long)b);
#else
  __builtin_memcpy(&x, &b, 8);
#endif
  return x;
}

}  // namespace emrkc_k
