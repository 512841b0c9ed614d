/*
 * emrkc.h — C ABI of the B200-native emRKC monodomain time step.
 *
 * This is the drop-in boundary for the reference's hot path
 * (arxiv/paper_2401_01745, /root/reference/proj). The reference binds its
 * integrators to the problem through std::function callbacks bundled in
 * `SplitRhs` (P/include/mrkc/multirate.hpp:25-35) and the virtual
 * `MonodomainProblem` / `IonicModel` interfaces
 * (P/include/mrkc/monodomain.hpp:93-176, P/include/mrkc/ionic.hpp:17-53).
 * Every entry point below replaces one reference function; the comment on
 * each names it (P/ = /root/reference/proj/).
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types cross the ABI.
 *  - State vectors use the reference `Vec` layout byte-for-byte:
 *    [V | gate_0 | ... | gate_{g-1} | aux_0 | ...], each block n_nodes long,
 *    node index i0 + n0*(i1 + n1*i2) (P/include/mrkc/monodomain.hpp:51-60,
 *    P/src/monodomain.cpp:36-44). With a partition, the blocks hold the
 *    local z-slab only (same layout, n_nodes = local node count).
 *  - Units are the reference's: mm, ms, mV, mS/mm, uF/mm^2, uA/mm^3.
 *  - Every function returns an emrkc_status. EMRKC_EINVAL maps to the
 *    reference's std::invalid_argument / ConfigError, EMRKC_ENONFINITE to
 *    NumericalAbort. emrkc_last_error() returns the message.
 *  - A handle owns one device and one CUDA stream; it is not thread-safe,
 *    distinct handles may be driven from distinct host threads.
 *  - There is no CPU fallback: every compute entry point runs sm_100a
 *    kernels and fails with EMRKC_ECUDA when no device is usable.
 */
#ifndef EMRKC_H
#define EMRKC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMRKC_ABI_VERSION 1

typedef enum emrkc_status {
  EMRKC_OK = 0,
  EMRKC_EINVAL = 1,     /* std::invalid_argument / ConfigError */
  EMRKC_ENONFINITE = 2, /* NumericalAbort (non-finite stage / norm guard) */
  EMRKC_ECUDA = 3,      /* CUDA runtime failure or no usable device */
  EMRKC_ESTATE = 4,     /* call out of order (e.g. no state uploaded) */
  EMRKC_ENOMEM = 5,
  EMRKC_ECALLBACK = 6   /* a caller-supplied device callback returned non-zero */
} emrkc_status;

enum { EMRKC_MODEL_HH = 0 };          /* make_ionic_model("hh"), P/src/ionic.cpp:125-128 */
/* SYNTHETIC width stand-in (SURVEY §8(c) option 2; no physiology claim): HH
 * plus n_aux passive auxiliary ("concentration-like") variables, so a state
 * has the CRN / TTP width N = 4 + n_aux (21 / 19) without their unavailable
 * equations. V and the gates follow HH exactly (the current ignores the aux
 * variables); aux a relaxes linearly towards a V-dependent target through
 * IonicModel::aux_rates (P/include/mrkc/ionic.hpp:33-36, f_S aux rows
 * P/src/monodomain.cpp:191-221):
 *   g_S,a = k_a * ((s1_a * V + s0_a) - z_a),
 *   k_a = 0.002 * (1 + a % 5), s1_a = 0.01 * (a % 3), s0_a = 0.5 + 0.1 * (a % 4),
 * evaluated in that order without FMA; rest: z_a = s1_a * V_rest + s0_a. */
enum { EMRKC_MODEL_HH_AUX = 1 };
#define EMRKC_MAX_AUX 20
/* SplitRhs::f_F / f_S; _GATES: f_F_with_gates / f_S_with_gates of the mRKC
 * stiff-gate split (P/src/monodomain.cpp:287-304, gates from
 * emrkc_set_stiff_gates) */
enum { EMRKC_RHS_F = 0, EMRKC_RHS_S = 1, EMRKC_RHS_F_GATES = 2, EMRKC_RHS_S_GATES = 3 };
/* EmrkcVariant, P/include/mrkc/multirate.hpp:37-40 (averaged force:
 * P/src/multirate.cpp:100-105 standard, :106-115 progressive). */
enum { EMRKC_VARIANT_STANDARD = 0, EMRKC_VARIANT_PROGRESSIVE = 1 };
enum {
  EMRKC_ABORT_NONE = 0,
  EMRKC_ABORT_NONFINITE = 1,  /* check_stage_finite, P/src/cheb.cpp:73-80 */
  EMRKC_ABORT_NORM_GUARD = 2  /* ||V||_inf > 1e6, P/src/simulate.cpp:222-227 */
};

/* Problem description. Replaces the arguments of
 * MonodomainOperator(Grid, Conductivity, IonicModel, StimulusProtocol)
 * (P/include/mrkc/monodomain.hpp:121-123) with plain data. The grid is
 * given by node counts (make_grid builds extent/dx + 1 nodes per axis,
 * P/src/monodomain.cpp:9-32; extent = (n-1)*dx here). */
typedef struct emrkc_problem {
  int32_t dim;                 /* 1, 2 or 3 */
  int32_t model;               /* EMRKC_MODEL_HH / EMRKC_MODEL_HH_AUX */
  int64_t n[3];                /* nodes per axis (1 on unused axes) */
  double dx[3];                /* [mm] */
  double sigma[3];             /* Conductivity::sigma [mS/mm] */
  double chi;                  /* [1/mm] */
  double C_m;                  /* [uF/mm^2] */
  double stim_chi_amplitude;   /* StimulusProtocol::chi_amplitude [uA/mm^3] */
  double stim_lo[3];           /* box_lo [mm] */
  double stim_hi[3];           /* box_hi [mm] */
  double stim_t0, stim_t1;     /* window [ms], inclusive */
  int32_t n_aux;               /* EMRKC_MODEL_HH_AUX: auxiliary variables (0 for HH) */
  int32_t reserved;
} emrkc_problem;

/* z-slab ownership along the slowest axis (axis dim-1). [z_begin, z_end).
 * A null partition means the whole grid. No reference counterpart: the
 * reference never partitions. */
typedef struct emrkc_partition {
  int64_t z_begin;
  int64_t z_end;
} emrkc_partition;

/* MultirateStepReport (P/include/mrkc/multirate.hpp:44-51) plus the abort
 * information the reference carries in NumericalAbort. */
typedef struct emrkc_step_report {
  int32_t s;            /* outer stages  (get_stages(dt, rho_S))      */
  int32_t m;            /* inner stages  (get_stages(eta, rho_F))     */
  double eta;           /* 2 dt / ell_s                                */
  double ell_s;
  double ell_m;
  int64_t n_fF;         /* EvalCounters deltas of this step            */
  int64_t n_fS;
  int64_t n_exp;
  int32_t abort_kind;   /* EMRKC_ABORT_*                               */
  int32_t abort_stage;  /* stage index named in the NumericalAbort msg */
  int32_t abort_inner;  /* 1: raised by the inner iteration            */
  int32_t abort_outer_stage; /* outer stage j in which it happened     */
} emrkc_step_report;

/* RunResult (P/include/mrkc/simulate.hpp:21-45) fields that the emRKC
 * branch of run_simulation fills (P/src/simulate.cpp:95-234). */
typedef struct emrkc_run_result {
  int64_t n_steps;      /* requested steps                              */
  int64_t steps_done;   /* steps whose result was accepted into y       */
  int32_t aborted;
  int32_t abort_kind;   /* EMRKC_ABORT_*                                */
  int64_t abort_step;   /* -1 when not aborted                          */
  int32_t abort_stage;
  int32_t abort_inner;
  double gate_min;      /* track_gate_range over the run                */
  double gate_max;
  int64_t n_fF;         /* EvalCounters                                  */
  int64_t n_fS;
  int64_t n_exp;
  int32_t s;            /* per-step plan (constant: rho is frozen)      */
  int32_t m;
  double eta;
  double device_ms;     /* CUDA-event time of the stepping loop         */
  int32_t abort_outer_stage; /* outer stage j of a non-finite abort     */
  int32_t reserved;
} emrkc_run_result;

/* RhoEstimate (P/include/mrkc/spectral.hpp:10-16). */
typedef struct emrkc_rho_result {
  double rho;           /* safety-multiplied estimate [1/ms] */
  int32_t iterations;
  int32_t converged;
  double safety;        /* 1.05 */
} emrkc_rho_result;

typedef struct emrkc_handle emrkc_handle;

/* ---- library / host-side numerics (no device needed) ------------------ */

const char* emrkc_version(void);

/* Thread-local message of the last failing call made without a handle
 * (or with a null handle); see also emrkc_last_error(). */
const char* emrkc_global_error(void);

/* get_stages(dt, rho, epsilon) — P/src/cheb.cpp:25-39. */
int emrkc_get_stages(double dt, double rho, double epsilon, int32_t* s,
                     double* ell, double* beta);

/* rkc_coeffs(s, epsilon) — P/src/cheb.cpp:41-69. Arrays have s+1 entries
 * (any may be null). */
int emrkc_rkc_coeffs(int32_t s, double epsilon, double* omega0,
                     double* omega1, double* b, double* mu, double* nu,
                     double* kappa, double* c);

/* plan_step (P/src/multirate.cpp:129-135): fills s, m, eta, ell_s, ell_m
 * and the per-step counters of *plan. */
int emrkc_plan_step(double dt, double rho_F, double rho_S, double epsilon,
                    emrkc_step_report* plan);

/* IonicModel::n_gates/n_aux — P/include/mrkc/ionic.hpp:22-23 (HH_AUX: the
 * aux count is per problem; the maximum, EMRKC_MAX_AUX, is reported). */
int emrkc_model_info(int32_t model, int32_t* n_gates, int32_t* n_aux);

/* IonicModel::resting_state — P/src/ionic.cpp:42-77. gates: n_gates. */
int emrkc_resting_state(int32_t model, double* V, double* gates);
/* MonodomainOperator::initial_state (P/src/monodomain.cpp:306-319): the
 * uniform resting state in Vec layout [V | gates | aux] (len = state len). */
int emrkc_initial_state(const emrkc_problem* p, double* y, int64_t len);

/* StateLayout::size() of the (local) state — P/include/mrkc/monodomain.hpp:56. */
int64_t emrkc_state_len(const emrkc_problem* p, const emrkc_partition* part);

/* Balanced z-slab split of n_z planes over nranks (uneven allowed). */
int emrkc_partition_slab(int64_t n_z, int32_t nranks, int32_t rank,
                         emrkc_partition* out);

/* ---- device handle ----------------------------------------------------- */

/* Builds the device operator: replaces constructing MonodomainOperator
 * (P/src/monodomain.cpp:305-311) and binding SplitRhs
 * (P/src/simulate.cpp:153-157). part may be null (whole grid). */
int emrkc_create(const emrkc_problem* p, int32_t device,
                 const emrkc_partition* part, emrkc_handle** out);
void emrkc_destroy(emrkc_handle* h);
const char* emrkc_last_error(const emrkc_handle* h);
int64_t emrkc_local_len(const emrkc_handle* h);

/* Upload / download the (local) state in reference Vec layout. */
int emrkc_set_state(emrkc_handle* h, const double* y, int64_t len);
int emrkc_get_state(emrkc_handle* h, double* y, int64_t len);
/* Kernel plan of the handle's current step plan (after a step / run):
 * 1 when one step runs as the single fused pass (k_fused2: s = 1, m = 2,
 * 3-D whole grid, EMRKC_FUSED=1 on a -DEMRKC_EXPERIMENTAL=1 build), 2 when it runs z-pipelined (node-kernel
 * chunks on the handle's stream, inner-stage chunks overlapping them on a
 * second stream, EMRKC_ZPIPE=K chunks), 3 when run loops fuse inner stage 2
 * of step n with the node update of step n + 1 (k_step_x, EMRKC_XSTEP=1), 0 when it runs as one launch per
 * stencil level. A diagnostic for benches and tests; no reference
 * counterpart. */
int32_t emrkc_fused_active(emrkc_handle* h);
/* Node kernel of the outer-stage level on this handle: 1 = k_node_pair (an
 * x-adjacent pair of nodes per thread; 3-D whole grids with HH proper on the
 * TMA path, EMRKC_PAIR=0 disables), 0 = k_node_tma or the family EMRKC_PIPE
 * selects. A diagnostic for benches and tests; no reference counterpart. */
int32_t emrkc_node_kernel(emrkc_handle* h);
/* Device pointer of the current state (valid until the next step/run). */
int emrkc_state_device_ptr(emrkc_handle* h, double** dptr);
int emrkc_synchronize(emrkc_handle* h);

/* MonodomainOperator::f_F / f_S (P/src/monodomain.cpp:207-221) and
 * exp_part (:246-256) on host buffers, evaluated on the device. Whole-grid
 * handles only. */
int emrkc_eval_rhs(emrkc_handle* h, int32_t which, double t,
                   const double* y, double* out, int64_t len);
int emrkc_exp_part(emrkc_handle* h, const double* y, double* lambda,
                   double* y_inf, int64_t len);

/* estimate_spectral_radius(t, y, f_F|f_S, v0, rho0) on the current state
 * (P/src/spectral.cpp:26-71). v0 null selects the reference's seeded
 * direction (mt19937_64(0x9e3779b97f4a7c15) U(-1,1), :16-22). v_out
 * (nullable) receives the final direction. Whole-grid handles only;
 * partitioned handles use emrkc_group_estimate_rho. */
int emrkc_estimate_rho(emrkc_handle* h, int32_t which, double t,
                       const double* v0, double rho0, emrkc_rho_result* out,
                       double* v_out);

/* rel_l2_error (P/src/monodomain.cpp:88-110: trapezoid-weighted L2 with
 * the quadrature weights :52-63) of SoA block `block` (0 = V, 1..3 the
 * gates) of the device state against `ref` (n_nodes values, host memory or,
 * with ref_on_device != 0, device memory). EMRKC_EINVAL if ||ref|| = 0.
 * Whole-grid handles. Reduction order differs from the reference's serial
 * sum (~1e-16 relative). */
int emrkc_rel_l2_error(emrkc_handle* h, int32_t block, const double* ref,
                       int32_t ref_on_device, double* out);

/* emrkc_step(t, y, dt, rhs, epsilon, variant, report)
 * (P/src/multirate.cpp:173-189) on the device-resident state. On a
 * non-finite stage it returns EMRKC_ENONFINITE, leaves the state
 * unchanged and fills report->abort_* (the NumericalAbort). */
int emrkc_step(emrkc_handle* h, double t, double dt, double epsilon,
               int32_t variant, double rho_F, double rho_S,
               emrkc_step_report* report);

/* emrkc_step over host buffers: the per-call drop-in of
 * `Vec emrkc_step(t, const Vec& y, ...)` — copies y in, steps, copies the
 * result out (y_out may alias y_in). One-launch steps (s = m = 1) stream
 * the state in z-chunks so the host->device copy, the step and the
 * device->host copy overlap (pinned host buffers make the copies
 * asynchronous). On EMRKC_ENONFINITE the device state is y_in and the
 * contents of y_out are unspecified (the reference throws: no result); when
 * y_out overlaps y_in the call is not pipelined and y_in is left untouched
 * on an abort, as the reference leaves y. */
int emrkc_step_host(emrkc_handle* h, double t, const double* y_in,
                    double* y_out, int64_t len, double dt, double epsilon,
                    int32_t variant, double rho_F, double rho_S,
                    emrkc_step_report* report);

/* The emRKC branch of run_simulation's stepping loop
 * (P/src/simulate.cpp:176-229): steps step0 .. step0+nsteps-1 with
 * t = step*dt, abort on non-finite stages, ||V||_inf > 1e6 guard and gate
 * range tracking — all on the device, with no per-step host sync. */
int emrkc_run(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt,
              double epsilon, int32_t variant, double rho_F, double rho_S,
              emrkc_run_result* res);

/* EXEX-RL, the reference's reference-solution stepper: Rush-Larsen gates
 * (exponential Euler with dt) and explicit Euler on V with the reaction
 * evaluated at the new gates — exex_rl_step, P/src/baselines.cpp:192-210,
 * with rush_larsen_update :89-128. One step of the device state; counters
 * n_fF = n_fS = n_exp = 1. exex_rl_step never throws NumericalAbort. */
int emrkc_exex_step(emrkc_handle* h, double t, double dt, emrkc_step_report* report);

/* run_simulation's exex_rl loop (P/src/simulate.cpp:164-165,176-229):
 * t = step*dt; the ||V||_inf > 1e6 guard (which also trips on a non-finite
 * V, max_abs_v :67-74) assigns the state and stops; gate range tracking.
 * res->s = res->m = 1, res->eta = dt. */
int emrkc_exex_run(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt,
                   emrkc_run_result* res);

/* mRKC with the stiff-gate split (run_simulation, P/src/simulate.cpp:132-150):
 * gates in `mask` (bit g = gate g; HH: 0 m, 1 h, 2 n) join f_F, the others
 * join f_S. Default mask 1 (m, the stiffest HH gate). */
int emrkc_set_stiff_gates(emrkc_handle* h, int32_t mask);
/* identify_stiff_gates (P/src/ionic.cpp:130-146): gates ordered by their
 * largest alpha + beta over the V samples (descending). order: n_gates. */
int emrkc_identify_stiff_gates(int32_t model, const double* V, int64_t n, int32_t* order);
/* mrkc_step (P/src/multirate.cpp:158-171, averaged force :60-76) on the
 * device state; rho_F / rho_S of f_F / f_S with gates (EMRKC_RHS_*_GATES).
 * Counters: n_fF = s m, n_fS = s, n_exp = 0. Whole-grid handles. */
int emrkc_mrkc_step(emrkc_handle* h, double t, double dt, double epsilon, double rho_F,
                    double rho_S, emrkc_step_report* report);
/* run_simulation's mrkc loop (P/src/simulate.cpp:191-195,176-229). */
int emrkc_mrkc_run(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt, double epsilon,
                   double rho_F, double rho_S, emrkc_run_result* res);

/* IMEX-RL (imex_rl_step, P/src/baselines.cpp:132-190): Rush-Larsen gates,
 * then (I - dt D) V = V + dt v_rhs by CG (cg_solve :20-82) in sqrt(w)-scaled
 * coordinates with the Jacobi preconditioner (jacobi != 0), relative
 * tolerance rel_tol (CgConfig default 1e-8) and max_iters (0: 10 sqrt(n)+1),
 * all on the device; *cg_iters (nullable) receives the CG iterations.
 * Counters: n_fF = iterations + 2, n_fS = n_exp = 1. A CG that does not
 * converge is the reference's NumericalAbort (EMRKC_ENONFINITE, stage -1). */
int emrkc_imex_step(emrkc_handle* h, double t, double dt, double rel_tol, int64_t max_iters,
                    int32_t jacobi, emrkc_step_report* report, int64_t* cg_iters);
/* run_simulation's imex_rl loop (P/src/simulate.cpp:164-165,176-229) with
 * CgConfig (rel_tol, max_iters, jacobi); *cg_iters_total (nullable) is
 * EvalCounters::cg_iters_total. */
int emrkc_imex_run(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt, double rel_tol,
                   int64_t max_iters, int32_t jacobi, emrkc_run_result* res,
                   int64_t* cg_iters_total);

/* Benchmark form of emrkc_run: before every step, writes flush_bytes of a
 * scratch buffer (evicts L2; 0 = no flush), then times every kernel launch
 * of the step with its own CUDA-event pair on the handle's stream.
 * launch_ms receives nsteps * s * m durations (launch order); the flush is
 * outside every timed pair. Same numerics and abort semantics as
 * emrkc_run; res->device_ms is the sum of the launch times. */
int emrkc_run_timed(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt,
                    double epsilon, int32_t variant, double rho_F,
                    double rho_S, int64_t flush_bytes, double* launch_ms,
                    int64_t launch_ms_len, emrkc_run_result* res);

/* ---- z-slab groups (multi-slab / multi-GPU) ---------------------------- */

/* A group steps the handles of consecutive z-slabs (ordered bottom to top)
 * in lockstep; V halo planes are written by each producing kernel straight
 * into the neighbour's ghost planes (peer stores over NVLink when the
 * neighbour lives on another device). Handles may share one device. */
typedef struct emrkc_group emrkc_group;
int emrkc_group_create(emrkc_handle* const* hs, int32_t n, emrkc_group** out);
void emrkc_group_destroy(emrkc_group* g);
int emrkc_group_estimate_rho(emrkc_group* g, int32_t which, double t,
                             emrkc_rho_result* out);
int emrkc_group_run(emrkc_group* g, int64_t step0, int64_t nsteps, double dt,
                    double epsilon, int32_t variant, double rho_F,
                    double rho_S, emrkc_run_result* res);

/* ---- multi-process (one process per GPU) ------------------------------- */

/* Cross-process ghost-plane link: each rank exports an opaque blob (CUDA
 * IPC handles of its ghost buffers and events), the host exchanges blobs
 * (e.g. torch.distributed all_gather_object), and each rank imports its
 * lower (side 0) and upper (side 1) neighbour's blob. */
int64_t emrkc_ipc_blob_size(void);
int emrkc_ipc_export(emrkc_handle* h, void* blob, int64_t len);
int emrkc_ipc_import(emrkc_handle* h, int32_t side, const void* blob,
                     int64_t len);
/* Local part of a distributed run: like emrkc_run, but the halo planes go
 * to the imported neighbours (peer stores from the producing kernel; the
 * neighbour's consuming blocks wait on a system-scope arrival counter, so
 * interior blocks never wait). Ranks do not fold abort words: the caller
 * reduces the per-rank results (first abort over ranks, min/max of gate
 * range) and, if a rank aborted, every rank calls emrkc_dist_replay for the
 * steps before the first abort (+1 for a norm-guard trip) to land on the
 * reference's final state. Needs the fast kernels. */
int emrkc_dist_run(emrkc_handle* h, int64_t step0, int64_t nsteps, double dt,
                   double epsilon, int32_t variant, double rho_F,
                   double rho_S, emrkc_run_result* res);
/* Restores the state the last emrkc_dist_run started from and runs nsteps
 * (collective: all ranks call it with the same arguments). */
int emrkc_dist_replay(emrkc_handle* h, int64_t step0, int64_t nsteps,
                      double dt, double epsilon, int32_t variant,
                      double rho_F, double rho_S, emrkc_run_result* res);

/* Testing aid for the distributed protocol on one process / one GPU:
 * link two adjacent slab handles directly (no IPC), then run all slabs with
 * every launch serialised (each device-side wait is satisfied when its
 * kernel starts, so no kernel ever waits on a concurrent one). replay != 0
 * restores the checkpoints first (emrkc_dist_replay semantics). */
int emrkc_dist_link_local(emrkc_handle* lower, emrkc_handle* upper);
int emrkc_dist_lockstep_run(emrkc_handle* const* hs, int32_t n, int32_t replay,
                            int64_t step0, int64_t nsteps, double dt,
                            double epsilon, int32_t variant, double rho_F,
                            double rho_S, emrkc_run_result* res);

/* Wide halo of the temporally blocked inner stages on slabs (north_star
 * (4); no reference counterpart — the reference never partitions). With
 * K = m - 1 inner stages fused into one pass (k_vin_tb, 2 <= K <= 4), a
 * slab needs K planes of d_1 from each neighbour: the inner-stage-1 kernel
 * stores its first / last K planes of d_1 straight into the neighbours' d_1
 * ghosts (peer stores, double-buffered by outer stage), and the fused pass
 * marches K planes into them. Only possible when every slab of the
 * partition is at least K planes deep, so the caller states the smallest
 * slab depth; every slab of a run must be given the same value
 * (emrkc_group_create and emrkc_dist_lockstep_run set it themselves). 0
 * (the default) keeps the per-stage inner kernels (one V plane per level). */
int emrkc_set_slab_min_depth(emrkc_handle* h, int64_t min_planes);

/* estimate_spectral_radius (P/src/spectral.cpp:26-71) over z-slabs held by
 * SEPARATE processes, one primitive at a time; the caller's host loop
 * (paper_2401_01745_b200/dist.py slab_rho) moves the V ghost planes between
 * ranks (any transport: NCCL send/recv of device planes) and chains the
 * norms across ranks. Chained in global order (SoA block by block, slabs in
 * z order, each slab continuing the running sum it received), the norms
 * are the reference's serial sums bit for bit, so rho does not depend on
 * the partition (SPEC: results independent of partitioning).
 *   begin : v := this slab's part of v0 (host slab; null: of the
 *           reference's seeded direction over the global state);
 *   plane : copy this slab's first (side 0) / last (side 1) V plane of
 *           field (0: v, 1: the state y) into device memory dst;
 *   sumsq : acc_out = acc_in + sum x^2 over SoA block `block` of field, in
 *           the reference's serial order;
 *   fy    : fy = f(t, y) with the neighbours' y ghost planes (device; null
 *           at the global boundary);
 *   step  : v := f(t, y + q v) - fy, with y and v ghosts;
 *   end   : copy the final direction (nullable) and release the work. */
int emrkc_slab_power_begin(emrkc_handle* h, int32_t which, const double* v0_slab);
int emrkc_slab_power_plane(emrkc_handle* h, int32_t field, int32_t side, double* dst);
int emrkc_slab_power_sumsq(emrkc_handle* h, int32_t field, int32_t block, double acc_in,
                           double* acc_out);
int emrkc_slab_power_fy(emrkc_handle* h, double t, const double* gy_lo, const double* gy_hi);
int emrkc_slab_power_step(emrkc_handle* h, double t, double q, const double* gy_lo,
                          const double* gy_hi, const double* gv_lo, const double* gv_hi);
int emrkc_slab_power_end(emrkc_handle* h, double* v_out_slab);

/* Testing aid for the cross-process (IPC) path with fewer GPUs than ranks:
 * when a hook is set, emrkc_dist_run / emrkc_dist_replay synchronise the
 * handle's stream after every stencil level and call hook(ctx) (e.g. a
 * host barrier across the ranks) before the next level, so every
 * device-side halo wait is already satisfied when its kernel starts and
 * ranks sharing one GPU never spin on each other. NULL clears it. */
typedef void (*emrkc_level_hook)(void* ctx);
int emrkc_set_level_hook(emrkc_handle* h, emrkc_level_hook hook, void* ctx);


/* ===========================================================================
 * The reference's integrator layer over DEVICE callbacks
 * (P/include/mrkc/cheb.hpp:60-63, multirate.hpp:19-35,57-81,
 * spectral.hpp:28-29). The reference's integrators are written against
 * std::function right-hand sides; here a right-hand side is a host
 * function that enqueues f(t, y) -> out on `stream` for DEVICE buffers y,
 * out of `len` doubles (the stream is a cudaStream_t). The recurrences,
 * exponential Euler updates, finite checks and power-iteration norms run in
 * sm_100a kernels on the context's stream, in the reference's operation
 * order; only the callbacks' own work is the caller's.
 * emrkc_bind_split_rhs() supplies callbacks bound to a handle's monodomain
 * operator (f_F, f_S, exp_part on its device kernels), so the generic layer
 * also runs the grid problem (the fused emrkc_step above is the fast path).
 * ======================================================================== */

/* RhsFn (P/include/mrkc/core.hpp:14) on device buffers. Non-zero return
 * aborts the caller with EMRKC_ECALLBACK. */
typedef int (*emrkc_rhs_fn)(void* ctx, double t, const double* y, double* out,
                            int64_t len, void* stream);
/* SplitRhs::exp_part (P/include/mrkc/multirate.hpp:29-31). */
typedef int (*emrkc_exp_part_fn)(void* ctx, const double* y, double* lambda,
                                 double* y_inf, int64_t len, void* stream);

/* EvalCounters (P/include/mrkc/core.hpp:34-57), the tallies the
 * integrators increment at their call sites (P/src/multirate.cpp:18-38). */
typedef struct emrkc_counters {
  int64_t n_fF;
  int64_t n_fS;
  int64_t n_exp_steps;
} emrkc_counters;

/* SplitRhs (P/include/mrkc/multirate.hpp:25-35). exp_part may be null
 * (mRKC); counters may be null. */
typedef struct emrkc_split_rhs {
  emrkc_rhs_fn f_F;
  void* f_F_ctx;
  emrkc_rhs_fn f_S;
  void* f_S_ctx;
  emrkc_exp_part_fn exp_part;
  void* exp_ctx;
  double rho_F;
  double rho_S;
  emrkc_counters* counters;
} emrkc_split_rhs;

/* A device + stream context for the generic layer (no problem attached). */
typedef struct emrkc_vctx emrkc_vctx;
int emrkc_vctx_create(int32_t device, emrkc_vctx** out);
void emrkc_vctx_destroy(emrkc_vctx* c);
const char* emrkc_vctx_last_error(const emrkc_vctx* c);
void* emrkc_vctx_stream(emrkc_vctx* c);  /* cudaStream_t of the context */
/* Device buffers on the context's device (stream-ordered allocator). */
int emrkc_vctx_alloc(emrkc_vctx* c, int64_t len, double** dptr);
int emrkc_vctx_free(emrkc_vctx* c, double* dptr);
int emrkc_vctx_upload(emrkc_vctx* c, double* dst, const double* host, int64_t len);
int emrkc_vctx_download(emrkc_vctx* c, double* host, const double* src, int64_t len);

/* exponential_euler_step(y, eta, lambda, y_inf) (P/src/multirate.cpp:49-58):
 * out = y + expm1(eta lambda) (y - y_inf), componentwise; device buffers
 * (out may alias y). */
int emrkc_exponential_euler(emrkc_vctx* c, const double* y, double eta,
                            const double* lambda, const double* y_inf,
                            int64_t len, double* out);

/* rkc_iteration(t, y, dt, f, s, epsilon) (P/src/cheb.cpp:84-105,
 * coefficients :41-69): the s-stage three-term recurrence over device
 * buffers, f evaluated exactly s times. A non-finite stage returns
 * EMRKC_ENONFINITE with *bad_stage = the stage index the reference's
 * NumericalAbort names (:73-80); out is then unspecified. */
int emrkc_rkc_iteration(emrkc_vctx* c, double t, const double* y, int64_t len,
                        double dt, emrkc_rhs_fn f, void* f_ctx, int32_t s,
                        double epsilon, double* out, int32_t* bad_stage);

/* averaged_force_emrkc (P/src/multirate.cpp:78-119; variant: standard
 * :100-105, progressive :106-115) and averaged_force_mrkc (:60-76):
 * out = (u_eta - y) / eta. *bad_stage as for emrkc_rkc_iteration (inner
 * stage). EMRKC_EINVAL for m < 1 or a missing exp_part (emRKC). */
int emrkc_averaged_force(emrkc_vctx* c, double t, const double* y, int64_t len,
                         double eta, const emrkc_split_rhs* rhs, int32_t m,
                         int32_t variant, double epsilon, double* out,
                         int32_t* bad_stage);
int emrkc_averaged_force_mrkc(emrkc_vctx* c, double t, const double* y,
                              int64_t len, double eta,
                              const emrkc_split_rhs* rhs, int32_t m,
                              double epsilon, double* out, int32_t* bad_stage);

/* emrkc_step(t, y, dt, rhs, epsilon, variant, report)
 * (P/src/multirate.cpp:173-189) and mrkc_step (:158-171) over a generic
 * SplitRhs: plan (s, eta, m) from rho_S / rho_F, outer rkc_iteration over
 * the averaged force. report (nullable) gets s, m, eta, ell_s, ell_m, the
 * counter deltas and, on EMRKC_ENONFINITE, the abort stage (abort_inner:
 * raised by an inner iteration). */
int emrkc_step_split(emrkc_vctx* c, double t, const double* y, int64_t len,
                     double dt, const emrkc_split_rhs* rhs, double epsilon,
                     int32_t variant, double* out, emrkc_step_report* report);
int emrkc_mrkc_step_split(emrkc_vctx* c, double t, const double* y,
                          int64_t len, double dt, const emrkc_split_rhs* rhs,
                          double epsilon, double* out,
                          emrkc_step_report* report);

/* estimate_spectral_radius(t, y, f, v0, rho0) (P/src/spectral.cpp:26-71)
 * over a generic device RhsFn: nonlinear power iteration with device
 * norms. v0 (device, nullable: the reference's seeded mt19937_64 direction,
 * :16-22), v_out (device, nullable) receives the final direction. */
int emrkc_estimate_spectral_radius(emrkc_vctx* c, double t, const double* y,
                                   int64_t len, emrkc_rhs_fn f, void* f_ctx,
                                   const double* v0, double rho0,
                                   emrkc_rho_result* out, double* v_out);

/* SplitRhs of a handle's MonodomainOperator (the binding of
 * P/src/simulate.cpp:153-157): f_F / f_S / exp_part callbacks on device
 * buffers of emrkc_local_len(h) doubles, run on the handle's kernels and
 * ordered after the caller's stream. rho_F / rho_S are left 0 (the caller
 * estimates them). Whole-grid handles only. */
int emrkc_bind_split_rhs(emrkc_handle* h, emrkc_split_rhs* out);

/* IonicModel (P/include/mrkc/ionic.hpp:17-53) pointwise formulas of a
 * model, host-side (setup / tests; the grid path evaluates them in the
 * kernels): rates(V) -> alpha, beta [n_gates]; ionic_current(V, z_E).
 * Bit-identical to the reference (P/src/ionic.cpp:14-40,98-116). */
int emrkc_model_rates(int32_t model, double V, double* alpha, double* beta);
int emrkc_model_ionic_current(int32_t model, double V, const double* z_E,
                              double* current);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* EMRKC_H */
