/*
 * emrkc_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's emRKC hot path
 * (arxiv/paper_2401_01745, /root/reference/proj = P/), used as the CPU
 * checker for the CUDA path and as the "port" CPU baseline. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline/reference legs may
 * load it; the product library never links or calls it.
 *
 * Parity of this restatement is pinned against the reference itself
 * (oracle/_ref/libmrkc_ref.so, compiled from the reference sources) and the
 * reference's own known-answer constants (tests/test_oracle_*.py).
 */
#ifndef EMRKC_ORACLE_H
#define EMRKC_ORACLE_H

#include <stdint.h>

#include "emrkc.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- cheb (P/src/cheb.cpp) --------------------------------------------- */
typedef struct oc_cheb {
  double value, derivative;
} oc_cheb;
oc_cheb oc_cheb_T(int degree, double x);
int oc_get_stages(double dt, double rho, double eps, int32_t* s, double* ell,
                  double* beta);
int oc_rkc_coeffs(int32_t s, double eps, double* omega0, double* omega1,
                  double* b, double* mu, double* nu, double* kappa, double* c);

/* generic callback RHS: out = f(t, y), n entries */
typedef void (*oc_rhs_fn)(void* ctx, double t, const double* y, double* out,
                          int64_t n);
typedef void (*oc_exp_fn)(void* ctx, const double* y, double* lam,
                          double* yinf, int64_t n);

typedef struct oc_counters {
  int64_t n_fF, n_fS, n_exp;
} oc_counters;

typedef struct oc_split {
  oc_rhs_fn f_F, f_S;
  oc_exp_fn exp_part;
  void* ctx;
  double rho_F, rho_S;
  oc_counters* counters; /* nullable */
} oc_split;

/* rkc_iteration (P/src/cheb.cpp:84-105). Returns 0 or EMRKC_ENONFINITE with
 * *abort_stage set. */
int oc_rkc_iteration(double t, const double* y, int64_t n, double dt,
                     oc_rhs_fn f, void* ctx, int32_t s, double eps,
                     double* out, int32_t* abort_stage);

/* ---- multirate (P/src/multirate.cpp) ----------------------------------- */
double oc_phi(double z);
void oc_exponential_euler_step(const double* y, double eta, const double* lam,
                               const double* yinf, int64_t n, double* out);
int oc_averaged_force_emrkc(double t, const double* y, int64_t n, double eta,
                            const oc_split* rhs, int32_t m, double eps,
                            double* out, int32_t* abort_stage);
int oc_emrkc_step(double t, const double* y, int64_t n, double dt,
                  const oc_split* rhs, double eps, double* out,
                  emrkc_step_report* rep);
/* variant: EMRKC_VARIANT_STANDARD / EMRKC_VARIANT_PROGRESSIVE */
int oc_emrkc_step_v(double t, const double* y, int64_t n, double dt,
                    const oc_split* rhs, double eps, int32_t variant,
                    double* out, emrkc_step_report* rep);

/* ---- HH ionic model (P/src/ionic.cpp) ----------------------------------- */
void oc_hh_rates(double V, double* alpha, double* beta);
void oc_hh_gate_coeffs(double V, double* lam, double* zinf);
double oc_hh_ionic_current(double V, const double* z);
int oc_hh_resting_state(double* V, double* gates);

/* ---- monodomain operator (P/src/monodomain.cpp) ------------------------ */
int64_t oc_state_len(const emrkc_problem* p);
int oc_validate(const emrkc_problem* p);
void oc_diffusion_apply(const emrkc_problem* p, const double* V, double* out);
double oc_stimulus_rate(const emrkc_problem* p, double t, int64_t node);
void oc_f_F(const emrkc_problem* p, double t, const double* y, double* out);
void oc_f_S(const emrkc_problem* p, double t, const double* y, double* out);
void oc_exp_part(const emrkc_problem* p, const double* y, double* lam,
                 double* yinf);
int oc_initial_state(const emrkc_problem* p, double* y);
double oc_rel_l2_error(const emrkc_problem* p, const double* a,
                       const double* b);
double oc_analytic_rho_F(const emrkc_problem* p);

/* ---- spectral (P/src/spectral.cpp) ------------------------------------- */
void oc_mt19937_64_uniform(uint64_t seed, int64_t n, double* out);
int oc_estimate_rho(const emrkc_problem* p, int32_t which, double t,
                    const double* y, const double* v0, double rho0,
                    emrkc_rho_result* out, double* v_out);
int oc_estimate_rho_cb(oc_rhs_fn f, void* ctx, int64_t n, double t,
                       const double* y, const double* v0, double rho0,
                       emrkc_rho_result* out, double* v_out);

/* ---- run loop (P/src/simulate.cpp:176-229, emRKC branch) --------------- */
int oc_run(const emrkc_problem* p, double* y, int64_t step0, int64_t nsteps,
           double dt, double eps, double rho_F, double rho_S,
           emrkc_run_result* res, double* wall_s);
/* Method (P/include/mrkc/config.hpp:17) of oc_run_method; OC_METHOD_MRKC
 * takes the stiff gate mask in bits 4..6 (oc_run_mrkc) */
enum { OC_METHOD_EMRKC = 0, OC_METHOD_EMRKC_PROGRESSIVE = 1, OC_METHOD_EXEX_RL = 2,
       OC_METHOD_MRKC = 3 };
/* internal variant code of oc_emrkc_step_v for mrkc_step (multirate.cpp:158-171) */
enum { OC_VARIANT_MRKC = 3 };
int oc_run_mrkc(const emrkc_problem* p, double* y, int64_t step0, int64_t nsteps,
                double dt, double eps, int32_t stiff, double rho_F, double rho_S,
                emrkc_run_result* res, double* wall_s);
/* f_F_with_gates / f_S_with_gates (P/src/monodomain.cpp:287-304), stiff gate mask */
void oc_f_F_gates(const emrkc_problem* p, int32_t stiff, double t, const double* y,
                  double* out);
void oc_f_S_gates(const emrkc_problem* p, int32_t stiff, double t, const double* y,
                  double* out);
/* imex_rl_step (P/src/baselines.cpp:132-190) and its run loop, CgConfig
 * (rel_tol, max_iters (0: 10 sqrt(n) + 1), jacobi) */
int oc_imex_rl_step(const emrkc_problem* p, double t, const double* y, double dt,
                    double rel_tol, int64_t max_iters, int32_t jacobi, double* out,
                    int64_t* iters, int64_t* applies);
int oc_run_imex(const emrkc_problem* p, double* y, int64_t step0, int64_t nsteps, double dt,
                double rel_tol, int64_t max_iters, int32_t jacobi, emrkc_run_result* res,
                int64_t* cg_iters_total);
/* identify_stiff_gates (P/src/ionic.cpp:130-146) for HH */
int oc_identify_stiff_gates(const double* V, int64_t n, int32_t* order);
int oc_run_method(const emrkc_problem* p, double* y, int64_t step0, int64_t nsteps,
                  double dt, double eps, int32_t method, double rho_F, double rho_S,
                  emrkc_run_result* res, double* wall_s);
/* exex_rl_step — P/src/baselines.cpp:192-210 (out: 4n, not aliasing y) */
int oc_exex_rl_step(const emrkc_problem* p, double t, const double* y, double dt,
                    double* out);
int oc_emrkc_step_grid(const emrkc_problem* p, double t, const double* y,
                       double dt, double eps, double rho_F, double rho_S,
                       double* out, emrkc_step_report* rep);

/* scalar surrogate split (P/tests/test_multirate.cpp:54-66) */
int oc_scalar_averaged_force(double lF, double lS, double lE, double yinf,
                             double y, double eta, int32_t m, double eps,
                             double* out);
int oc_scalar_emrkc_step(double lF, double lS, double lE, double yinf,
                         double y, double dt, double eps, double* out,
                         int32_t* s, int32_t* m, double* eta);

const char* oc_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
