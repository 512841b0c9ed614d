/*
 * emrkc_oracle.c — TEST INFRASTRUCTURE ONLY (CPU checker; see header).
 *
 * Plain-C restatement of the reference's emRKC path. Each function cites the
 * reference file:line it restates (P/ = /root/reference/proj/). Floating-point
 * operations are written in the reference's evaluation order so that, built
 * with the same (non-FMA, non-fast-math) x86-64 code generation and the same
 * libm, results are bit-identical to the reference; tests pin that against
 * oracle/_ref/libmrkc_ref.so.
 */
#define _POSIX_C_SOURCE 200809L
#include "emrkc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* oc_last_error(void) { return g_err; }

/* ======================= cheb (P/src/cheb.cpp) ======================== */

/* cheb_T — P/src/cheb.cpp:8-23 */
oc_cheb oc_cheb_T(int degree, double x) {
  double tm1 = 1.0, dm1 = 0.0;
  oc_cheb r = {tm1, dm1};
  if (degree <= 0) return r;
  double t = x, d = 1.0;
  for (int j = 2; j <= degree; ++j) {
    const double tj = 2.0 * x * t - tm1;
    const double dj = 2.0 * t + 2.0 * x * d - dm1;
    tm1 = t;
    dm1 = d;
    t = tj;
    d = dj;
  }
  r.value = t;
  r.derivative = d;
  return r;
}

/* get_stages — P/src/cheb.cpp:25-39 */
int oc_get_stages(double dt, double rho, double eps, int32_t* s, double* ell,
                  double* beta) {
  if (!isfinite(dt) || !isfinite(rho) || !isfinite(eps))
    return fail(EMRKC_EINVAL, "get_stages: non-finite input");
  if (dt <= 0.0) return fail(EMRKC_EINVAL, "get_stages: dt must be > 0");
  if (rho < 0.0) return fail(EMRKC_EINVAL, "get_stages: rho must be >= 0");
  if (eps < 0.0 || eps >= 1.5)
    return fail(EMRKC_EINVAL, "get_stages: damping must be in [0, 1.5)");
  const double b = 2.0 - 4.0 * eps / 3.0;
  const int si = (int)ceil(sqrt(dt * rho / b));
  const int ss = si > 1 ? si : 1;
  *s = ss;
  *ell = b * (double)ss * ss;
  *beta = b;
  return 0;
}

/* rkc_coeffs — P/src/cheb.cpp:41-69 */
int oc_rkc_coeffs(int32_t s, double eps, double* omega0, double* omega1,
                  double* b, double* mu, double* nu, double* kappa,
                  double* c) {
  if (s < 1) return fail(EMRKC_EINVAL, "rkc_coeffs: s must be >= 1");
  const double w0 = 1.0 + eps / ((double)s * s);
  const oc_cheb ts = oc_cheb_T(s, w0);
  const double w1 = ts.value / ts.derivative;
  for (int j = 0; j <= s; ++j) {
    b[j] = 1.0 / oc_cheb_T(j, w0).value;
    mu[j] = nu[j] = kappa[j] = c[j] = 0.0;
  }
  mu[1] = w1 / w0;
  c[0] = 0.0;
  c[1] = mu[1];
  for (int j = 2; j <= s; ++j) {
    mu[j] = 2.0 * w1 * b[j] / b[j - 1];
    nu[j] = 2.0 * w0 * b[j] / b[j - 1];
    kappa[j] = -b[j] / b[j - 2];
    c[j] = nu[j] * c[j - 1] + kappa[j] * c[j - 2] + mu[j];
  }
  *omega0 = w0;
  *omega1 = w1;
  return 0;
}

typedef struct coeffs {
  int s;
  double w0, w1;
  double *b, *mu, *nu, *kappa, *c;
} coeffs;

static int coeffs_make(coeffs* k, int s, double eps) {
  k->s = s;
  double* mem = (double*)calloc(5 * (size_t)(s + 1), sizeof(double));
  if (!mem) return fail(EMRKC_ENOMEM, "out of memory");
  k->b = mem;
  k->mu = mem + (s + 1);
  k->nu = mem + 2 * (s + 1);
  k->kappa = mem + 3 * (s + 1);
  k->c = mem + 4 * (s + 1);
  const int rc = oc_rkc_coeffs(s, eps, &k->w0, &k->w1, k->b, k->mu, k->nu,
                               k->kappa, k->c);
  if (rc) free(mem);
  return rc;
}
static void coeffs_free(coeffs* k) { free(k->b); }

/* check_stage_finite — P/src/cheb.cpp:73-80 */
static int stage_finite(const double* g, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(g[i])) return 0;
  return 1;
}

/* rkc_iteration — P/src/cheb.cpp:84-105. Three work vectors plus fbuf. */
static int rkc_iteration_k(double t, const double* y, int64_t n, double dt,
                           oc_rhs_fn f, void* ctx, const coeffs* k,
                           double* out, int32_t* abort_stage) {
  double* fbuf = (double*)malloc(sizeof(double) * n);
  double* gm2 = (double*)malloc(sizeof(double) * n);
  double* gm1 = (double*)malloc(sizeof(double) * n);
  int rc = 0;
  if (!fbuf || !gm2 || !gm1) {
    rc = fail(EMRKC_ENOMEM, "out of memory");
    goto done;
  }
  f(ctx, t, y, fbuf, n);
  memcpy(gm2, y, sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) gm1[i] = y[i] + k->mu[1] * dt * fbuf[i];
  if (!stage_finite(gm1, n)) {
    *abort_stage = 1;
    rc = fail(EMRKC_ENONFINITE, "rkc_iteration: non-finite value at stage 1");
    goto done;
  }
  for (int j = 2; j <= k->s; ++j) {
    f(ctx, t + k->c[j - 1] * dt, gm1, fbuf, n);
    for (int64_t i = 0; i < n; ++i)
      gm2[i] = k->nu[j] * gm1[i] + k->kappa[j] * gm2[i] +
               k->mu[j] * dt * fbuf[i];
    double* tmp = gm1;
    gm1 = gm2;
    gm2 = tmp;
    if (!stage_finite(gm1, n)) {
      *abort_stage = j;
      snprintf(g_err, sizeof g_err,
               "rkc_iteration: non-finite value at stage %d", j);
      rc = EMRKC_ENONFINITE;
      goto done;
    }
  }
  memcpy(out, gm1, sizeof(double) * n);
done:
  free(fbuf);
  free(gm2);
  free(gm1);
  return rc;
}

int oc_rkc_iteration(double t, const double* y, int64_t n, double dt,
                     oc_rhs_fn f, void* ctx, int32_t s, double eps,
                     double* out, int32_t* abort_stage) {
  coeffs k;
  int rc = coeffs_make(&k, s, eps);
  if (rc) return rc;
  rc = rkc_iteration_k(t, y, n, dt, f, ctx, &k, out, abort_stage);
  coeffs_free(&k);
  return rc;
}

/* ===================== multirate (P/src/multirate.cpp) ================== */

/* phi — P/src/multirate.cpp:42-47 */
double oc_phi(double z) {
  if (fabs(z) < 1e-5) return 1.0 + z * (0.5 + z * (1.0 / 6.0 + z / 24.0));
  return expm1(z) / z;
}

/* exponential_euler_step — P/src/multirate.cpp:49-58 */
void oc_exponential_euler_step(const double* y, double eta, const double* lam,
                               const double* yinf, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i)
    out[i] = y[i] + expm1(eta * lam[i]) * (y[i] - yinf[i]);
}

/* f_u(r, u) = f_F(r, u) + fs — P/src/multirate.cpp:101-104 */
typedef struct fu_ctx {
  const oc_split* rhs;
  const double* fs;
  const double* expc; /* progressive variant: (y_E - y)/eta, else NULL */
} fu_ctx;

static void f_u(void* vctx, double r, const double* u, double* out,
                int64_t n) {
  fu_ctx* c = (fu_ctx*)vctx;
  c->rhs->f_F(c->rhs->ctx, r, u, out, n);
  if (c->rhs->counters) ++c->rhs->counters->n_fF;
  if (c->expc) /* P/src/multirate.cpp:111-112 */
    for (int64_t i = 0; i < n; ++i) out[i] += c->fs[i] + c->expc[i];
  else /* :101-103 */
    for (int64_t i = 0; i < n; ++i) out[i] += c->fs[i];
}

/* averaged_force_emrkc — P/src/multirate.cpp:78-119 (standard :100-105,
 * progressive :106-115) */
static int averaged_force_k(double t, const double* y, int64_t n, double eta,
                            const oc_split* rhs, const coeffs* km, int32_t variant,
                            double* out, int32_t* abort_stage) {
  double* lam = (double*)malloc(sizeof(double) * n);
  double* yinf = (double*)malloc(sizeof(double) * n);
  double* yE = (double*)malloc(sizeof(double) * n);
  double* fs = (double*)malloc(sizeof(double) * n);
  double* expc = NULL;
  int rc = 0;
  if (!lam || !yinf || !yE || !fs) {
    rc = fail(EMRKC_ENOMEM, "out of memory");
    goto done;
  }
  rhs->exp_part(rhs->ctx, y, lam, yinf, n);
  oc_exponential_euler_step(y, eta, lam, yinf, n, yE);
  if (rhs->counters) ++rhs->counters->n_exp;
  rhs->f_S(rhs->ctx, t, yE, fs, n); /* slow term frozen at y_E (:96-97) */
  if (rhs->counters) ++rhs->counters->n_fS;
  if (variant == EMRKC_VARIANT_STANDARD) {
    fu_ctx c = {rhs, fs, NULL};
    rc = rkc_iteration_k(t, yE, n, eta, f_u, &c, km, out, abort_stage);
  } else {
    /* phi(eta Lambda) f_E(y) = (y_E - y)/eta (:107-109); iterate from y */
    expc = (double*)malloc(sizeof(double) * n);
    if (!expc) {
      rc = fail(EMRKC_ENOMEM, "out of memory");
      goto done;
    }
    for (int64_t i = 0; i < n; ++i) expc[i] = (yE[i] - y[i]) / eta;
    fu_ctx c = {rhs, fs, expc};
    rc = rkc_iteration_k(t, y, n, eta, f_u, &c, km, out, abort_stage);
  }
  if (rc) goto done;
  for (int64_t i = 0; i < n; ++i) out[i] = (out[i] - y[i]) / eta; /* :117 */
done:
  free(lam);
  free(yinf);
  free(yE);
  free(fs);
  free(expc);
  return rc;
}

/* averaged_force_mrkc — P/src/multirate.cpp:60-76: slow term frozen at y,
 * inner RKC from y on f_F + fs */
static int averaged_force_mrkc_k(double t, const double* y, int64_t n, double eta,
                                 const oc_split* rhs, const coeffs* km, double* out,
                                 int32_t* abort_stage) {
  double* fs = (double*)malloc(sizeof(double) * n);
  if (!fs) return fail(EMRKC_ENOMEM, "out of memory");
  rhs->f_S(rhs->ctx, t, y, fs, n);
  if (rhs->counters) ++rhs->counters->n_fS;
  fu_ctx c = {rhs, fs, NULL};
  int rc = rkc_iteration_k(t, y, n, eta, f_u, &c, km, out, abort_stage);
  if (!rc)
    for (int64_t i = 0; i < n; ++i) out[i] = (out[i] - y[i]) / eta; /* :74 */
  free(fs);
  return rc;
}

int oc_averaged_force_emrkc(double t, const double* y, int64_t n, double eta,
                            const oc_split* rhs, int32_t m, double eps,
                            double* out, int32_t* abort_stage) {
  if (m < 1) return fail(EMRKC_EINVAL, "averaged_force_emrkc: m must be >= 1");
  if (!rhs->exp_part)
    return fail(EMRKC_EINVAL, "averaged_force_emrkc: exp_part missing");
  coeffs km;
  int rc = coeffs_make(&km, m, eps);
  if (rc) return rc;
  rc = averaged_force_k(t, y, n, eta, rhs, &km, EMRKC_VARIANT_STANDARD, out, abort_stage);
  coeffs_free(&km);
  return rc;
}

/* the outer RKC iteration's right-hand side: the averaged force
 * (P/src/multirate.cpp:183-185) */
typedef struct avg_ctx {
  const oc_split* rhs;
  const coeffs* km;
  double eta;
  int rc;
  int32_t inner_stage;
  int32_t variant;
} avg_ctx;

static void f_avg(void* vctx, double r, const double* g, double* out,
                  int64_t n) {
  avg_ctx* c = (avg_ctx*)vctx;
  if (c->rc) { /* a previous inner iteration already aborted */
    for (int64_t i = 0; i < n; ++i) out[i] = NAN;
    return;
  }
  int32_t st = 0;
  c->rc = c->variant == OC_VARIANT_MRKC
              ? averaged_force_mrkc_k(r, g, n, c->eta, c->rhs, c->km, out, &st)
              : averaged_force_k(r, g, n, c->eta, c->rhs, c->km, c->variant, out, &st);
  if (c->rc) {
    c->inner_stage = st;
    for (int64_t i = 0; i < n; ++i) out[i] = NAN;
  }
}

int oc_emrkc_step(double t, const double* y, int64_t n, double dt,
                  const oc_split* rhs, double eps, double* out,
                  emrkc_step_report* rep) {
  return oc_emrkc_step_v(t, y, n, dt, rhs, eps, EMRKC_VARIANT_STANDARD, out, rep);
}

/* emrkc_step — P/src/multirate.cpp:173-189 with plan_step :129-135 */
int oc_emrkc_step_v(double t, const double* y, int64_t n, double dt,
                    const oc_split* rhs, double eps, int32_t variant,
                    double* out, emrkc_step_report* rep) {
  memset(rep, 0, sizeof(*rep));
  if (variant != EMRKC_VARIANT_STANDARD && variant != EMRKC_VARIANT_PROGRESSIVE &&
      variant != OC_VARIANT_MRKC)
    return fail(EMRKC_EINVAL, "emrkc_step: unknown variant");
  if (dt <= 0.0) return fail(EMRKC_EINVAL, "emrkc_step: dt must be > 0");
  /* mrkc_step (P/src/multirate.cpp:158-171) needs no exp_part */
  if (!rhs->exp_part && variant != OC_VARIANT_MRKC)
    return fail(EMRKC_EINVAL, "emrkc_step: exp_part missing");
  int32_t s, m;
  double ell_s, ell_m, beta;
  int rc = oc_get_stages(dt, rhs->rho_S, eps, &s, &ell_s, &beta);
  if (rc) return rc;
  const double eta = 2.0 * dt / ell_s;
  rc = oc_get_stages(eta, rhs->rho_F, eps, &m, &ell_m, &beta);
  if (rc) return rc;
  rep->s = s;
  rep->m = m;
  rep->eta = eta;
  rep->ell_s = ell_s;
  rep->ell_m = ell_m;
  oc_counters before = {0, 0, 0};
  if (rhs->counters) before = *rhs->counters;

  coeffs ks, km;
  if ((rc = coeffs_make(&ks, s, eps))) return rc;
  if ((rc = coeffs_make(&km, m, eps))) {
    coeffs_free(&ks);
    return rc;
  }
  avg_ctx c = {rhs, &km, eta, 0, 0, variant};
  int32_t outer_stage = 0;
  /* The reference throws out of the inner iteration at the first
   * non-finite inner stage; emulate by running the outer iteration stage by
   * stage and stopping at the first failure (inner before outer check). */
  double* fbuf = (double*)malloc(sizeof(double) * n);
  double* gm2 = (double*)malloc(sizeof(double) * n);
  double* gm1 = (double*)malloc(sizeof(double) * n);
  if (!fbuf || !gm2 || !gm1) {
    rc = fail(EMRKC_ENOMEM, "out of memory");
    goto done;
  }
  /* rkc_iteration (P/src/cheb.cpp:84-105) over the averaged force */
  f_avg(&c, t, y, fbuf, n);
  if (c.rc) {
    outer_stage = 1;
    goto aborted;
  }
  memcpy(gm2, y, sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) gm1[i] = y[i] + ks.mu[1] * dt * fbuf[i];
  if (!stage_finite(gm1, n)) {
    outer_stage = 1;
    goto aborted_outer;
  }
  for (int j = 2; j <= s; ++j) {
    f_avg(&c, t + ks.c[j - 1] * dt, gm1, fbuf, n);
    if (c.rc) {
      outer_stage = j;
      goto aborted;
    }
    for (int64_t i = 0; i < n; ++i)
      gm2[i] = ks.nu[j] * gm1[i] + ks.kappa[j] * gm2[i] +
               ks.mu[j] * dt * fbuf[i];
    double* tmp = gm1;
    gm1 = gm2;
    gm2 = tmp;
    if (!stage_finite(gm1, n)) {
      outer_stage = j;
      goto aborted_outer;
    }
  }
  memcpy(out, gm1, sizeof(double) * n);
  goto done;
aborted:
  rc = c.rc;
  rep->abort_kind = EMRKC_ABORT_NONFINITE;
  rep->abort_stage = c.inner_stage;
  rep->abort_inner = 1;
  rep->abort_outer_stage = outer_stage;
  goto done;
aborted_outer:
  rc = EMRKC_ENONFINITE;
  snprintf(g_err, sizeof g_err, "rkc_iteration: non-finite value at stage %d",
           outer_stage);
  rep->abort_kind = EMRKC_ABORT_NONFINITE;
  rep->abort_stage = outer_stage;
  rep->abort_inner = 0;
  rep->abort_outer_stage = outer_stage;
done:
  if (rhs->counters) {
    rep->n_fF = rhs->counters->n_fF - before.n_fF;
    rep->n_fS = rhs->counters->n_fS - before.n_fS;
    rep->n_exp = rhs->counters->n_exp - before.n_exp;
  }
  free(fbuf);
  free(gm2);
  free(gm1);
  coeffs_free(&ks);
  coeffs_free(&km);
  return rc;
}

/* ==================== HH ionic model (P/src/ionic.cpp) ================== */

/* lin_exp_ratio — P/src/ionic.cpp:14-21 */
static double lin_exp_ratio(double x, double k) {
  const double u = x / k;
  if (fabs(u) < 1e-4) return k * (1.0 + u * (0.5 + u / 12.0));
  return x / (1.0 - exp(-u));
}

/* HodgkinHuxley::rates — P/src/ionic.cpp:98-109 */
void oc_hh_rates(double V, double* alpha, double* beta) {
  alpha[0] = 0.1 * lin_exp_ratio(V + 40.0, 10.0);
  beta[0] = 4.0 * exp(-(V + 65.0) / 18.0);
  alpha[1] = 0.07 * exp(-(V + 65.0) / 20.0);
  beta[1] = 1.0 / (1.0 + exp(-(V + 35.0) / 10.0));
  alpha[2] = 0.01 * lin_exp_ratio(V + 55.0, 10.0);
  beta[2] = 0.125 * exp(-(V + 65.0) / 80.0);
}

/* IonicModel::gate_coeffs — P/src/ionic.cpp:31-40 */
void oc_hh_gate_coeffs(double V, double* lam, double* zinf) {
  double a[3], b[3];
  oc_hh_rates(V, a, b);
  for (int g = 0; g < 3; ++g) {
    lam[g] = -(a[g] + b[g]);
    zinf[g] = a[g] / (a[g] + b[g]);
  }
}

/* HodgkinHuxley::ionic_current — P/src/ionic.cpp:111-116, constants :86-91 */
double oc_hh_ionic_current(double V, const double* z) {
  const double m = z[0], h = z[1], n = z[2];
  return 1.2 * m * m * m * h * (V - 50.0) + 0.36 * n * n * n * n * (V - -77.0) +
         0.003 * (V - -54.387);
}

static double steady_current(double V) {
  double lam[3], zinf[3];
  oc_hh_gate_coeffs(V, lam, zinf);
  return oc_hh_ionic_current(V, zinf);
}

/* IonicModel::resting_state — P/src/ionic.cpp:42-77 */
int oc_hh_resting_state(double* V, double* gates) {
  double lo = -90.0, hi = -40.0;
  double flo = steady_current(lo), fhi = steady_current(hi);
  if (flo * fhi > 0.0)
    return fail(EMRKC_EINVAL, "resting_state: no sign change in [-90, -40] mV");
  for (int it = 0; it < 200 && hi - lo > 1e-14; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double fm = steady_current(mid);
    if (flo * fm <= 0.0) {
      hi = mid;
      fhi = fm;
    } else {
      lo = mid;
      flo = fm;
    }
  }
  (void)fhi;
  *V = 0.5 * (lo + hi);
  double lam[3];
  oc_hh_gate_coeffs(*V, lam, gates);
  return 0;
}

/* ================ monodomain operator (P/src/monodomain.cpp) ============ */

static int64_t n_nodes(const emrkc_problem* p) {
  int64_t nn = 1;
  for (int a = 0; a < p->dim; ++a) nn *= p->n[a];
  return nn;
}

/* auxiliary variables of the SYNTHETIC width stand-in EMRKC_MODEL_HH_AUX
 * (include/emrkc.h; the reference runs it through oracle/ref_driver.cpp's
 * HHAux IonicModel) */
static int n_aux_of(const emrkc_problem* p) {
  return p->model == EMRKC_MODEL_HH_AUX ? p->n_aux : 0;
}
static double aux_k(int a) { return 0.002 * (double)(1 + a % 5); }
static double aux_s1(int a) { return 0.01 * (double)(a % 3); }
static double aux_s0(int a) { return 0.5 + 0.1 * (double)(a % 4); }

int64_t oc_state_len(const emrkc_problem* p) { return n_nodes(p) * (4 + n_aux_of(p)); }

int oc_validate(const emrkc_problem* p) {
  if (p->dim < 1 || p->dim > 3)
    return fail(EMRKC_EINVAL, "grid: dim must be 1, 2, or 3");
  if (p->model != EMRKC_MODEL_HH && p->model != EMRKC_MODEL_HH_AUX)
    return fail(EMRKC_EINVAL, "unknown ionic model");
  if (p->model == EMRKC_MODEL_HH_AUX && (p->n_aux < 1 || p->n_aux > EMRKC_MAX_AUX))
    return fail(EMRKC_EINVAL, "hh_aux: n_aux out of range");
  for (int a = 0; a < p->dim; ++a)
    if (p->n[a] < 2 || !(p->dx[a] > 0.0))
      return fail(EMRKC_EINVAL, "grid: extent and dx must be positive");
  return 0;
}

static int64_t axis_stride(const emrkc_problem* p, int axis) {
  int64_t s = 1;
  for (int a = 0; a < axis; ++a) s *= p->n[a];
  return s;
}

/* diffusion_apply — P/src/monodomain.cpp:73-90 */
void oc_diffusion_apply(const emrkc_problem* p, const double* V, double* out) {
  const int64_t nn = n_nodes(p);
  for (int64_t i = 0; i < nn; ++i) out[i] = 0.0;
  for (int a = 0; a < p->dim; ++a) {
    const double w = p->sigma[a] / (p->chi * p->C_m * p->dx[a] * p->dx[a]);
    const int64_t stride = axis_stride(p, a);
    const int64_t na = p->n[a];
    for (int64_t i = 0; i < nn; ++i) {
      const int64_t ia = (i / stride) % na;
      const double vm = (ia > 0) ? V[i - stride] : V[i + stride];
      const double vp = (ia < na - 1) ? V[i + stride] : V[i - stride];
      out[i] += w * (vp - 2.0 * V[i] + vm);
    }
  }
}

/* stimulus_rate — P/src/monodomain.cpp:151-158, node_coord :48-50,
 * StimulusProtocol::active_at P/include/mrkc/monodomain.hpp:71 */
double oc_stimulus_rate(const emrkc_problem* p, double t, int64_t node) {
  if (p->stim_chi_amplitude == 0.0 || !(t >= p->stim_t0 && t <= p->stim_t1))
    return 0.0;
  for (int a = 0; a < p->dim; ++a) {
    const int64_t ia = (node / axis_stride(p, a)) % p->n[a];
    const double x = (double)ia * p->dx[a];
    if (x < p->stim_lo[a] - 1e-12 || x > p->stim_hi[a] + 1e-12) return 0.0;
  }
  return p->stim_chi_amplitude / (p->chi * p->C_m);
}

/* f_F — P/src/monodomain.cpp:207-212 */
void oc_f_F(const emrkc_problem* p, double t, const double* y, double* out) {
  (void)t;
  const int64_t nn = n_nodes(p), len = oc_state_len(p);
  for (int64_t k = nn; k < len; ++k) out[k] = 0.0;
  oc_diffusion_apply(p, y, out);
}

/* f_S — P/src/monodomain.cpp:214-221 -> v_reaction :160-173, aux rows
 * aux_rates_field :191-205 */
void oc_f_S(const emrkc_problem* p, double t, const double* y, double* out) {
  const int64_t nn = n_nodes(p), len = oc_state_len(p);
  const int na = n_aux_of(p);
  for (int64_t k = nn; k < len; ++k) out[k] = 0.0;
  for (int64_t i = 0; i < nn; ++i) {
    const double z[3] = {y[nn + i], y[2 * nn + i], y[3 * nn + i]};
    out[i] = oc_stimulus_rate(p, t, i) - oc_hh_ionic_current(y[i], z) / p->C_m;
    for (int a = 0; a < na; ++a) {
      const int64_t k = (4 + a) * nn + i;
      out[k] = aux_k(a) * ((aux_s1(a) * y[i] + aux_s0(a)) - y[k]);
    }
  }
}

/* exp_part — P/src/monodomain.cpp:246-256 -> gate_coeffs_field :175-189 */
void oc_exp_part(const emrkc_problem* p, const double* y, double* lam,
                 double* yinf) {
  const int64_t nn = n_nodes(p), len = oc_state_len(p);
  for (int64_t k = 0; k < len; ++k) lam[k] = yinf[k] = 0.0;
  for (int64_t i = 0; i < nn; ++i) {
    double l[3], zi[3];
    oc_hh_gate_coeffs(y[i], l, zi);
    for (int g = 0; g < 3; ++g) {
      lam[(1 + g) * nn + i] = l[g];
      yinf[(1 + g) * nn + i] = zi[g];
    }
  }
}

/* initial_state — P/src/monodomain.cpp:306-319 */
int oc_initial_state(const emrkc_problem* p, double* y) {
  double V, z[3];
  const int rc = oc_hh_resting_state(&V, z);
  if (rc) return rc;
  const int64_t nn = n_nodes(p);
  for (int64_t i = 0; i < nn; ++i) y[i] = V;
  for (int g = 0; g < 3; ++g)
    for (int64_t i = 0; i < nn; ++i) y[(1 + g) * nn + i] = z[g];
  for (int a = 0; a < n_aux_of(p); ++a) { /* HHAux::resting_state */
    const double za = aux_s1(a) * V + aux_s0(a);
    for (int64_t i = 0; i < nn; ++i) y[(4 + a) * nn + i] = za;
  }
  return 0;
}

/* quadrature_weights + l2_norm + rel_l2_error — P/src/monodomain.cpp:52-110 */
static double l2_norm_w(const emrkc_problem* p, const double* u) {
  const int64_t nn = n_nodes(p);
  double cell = 1.0;
  for (int a = 0; a < p->dim; ++a) cell *= p->dx[a];
  double s = 0.0;
  for (int64_t i = 0; i < nn; ++i) {
    double w = 1.0;
    for (int a = 0; a < p->dim; ++a) {
      const int64_t ia = (i / axis_stride(p, a)) % p->n[a];
      if (ia == 0 || ia == p->n[a] - 1) w *= 0.5;
    }
    s += w * u[i] * u[i];
  }
  return sqrt(cell * s);
}

double oc_rel_l2_error(const emrkc_problem* p, const double* a,
                       const double* b) {
  const int64_t nn = n_nodes(p);
  double* d = (double*)malloc(sizeof(double) * nn);
  if (!d) return NAN;
  for (int64_t i = 0; i < nn; ++i) d[i] = a[i] - b[i];
  const double nb = l2_norm_w(p, b);
  double r = NAN;
  if (nb != 0.0) r = l2_norm_w(p, d) / nb;
  free(d);
  return r;
}

/* analytic_rho_F — P/src/monodomain.cpp:112-121 */
double oc_analytic_rho_F(const emrkc_problem* p) {
  const double pi = 3.14159265358979323846;
  double rho = 0.0;
  for (int a = 0; a < p->dim; ++a) {
    const double w = p->sigma[a] / (p->chi * p->C_m * p->dx[a] * p->dx[a]);
    const double na = (double)p->n[a];
    const double s = sin((na - 1.0) * pi / (2.0 * na));
    rho += 4.0 * w * s * s;
  }
  return rho;
}

/* ======================= spectral (P/src/spectral.cpp) ================== */

/* std::mt19937_64 (the published MT19937-64 recurrence) feeding
 * std::uniform_real_distribution<double>(-1, 1) as libstdc++ implements it:
 * generate_canonical<double, 53> takes one 64-bit draw, x / 2^64 (clamped
 * below 1), then a + (b - a) * u. Restates seeded_direction,
 * P/src/spectral.cpp:16-22. */
void oc_mt19937_64_uniform(uint64_t seed, int64_t n, double* out) {
  enum { NN = 312, MM = 156 };
  const uint64_t A = 0xB5026F5AA96619E9ULL, UM = 0xFFFFFFFF80000000ULL,
                 LM = 0x7FFFFFFFULL;
  uint64_t mt[NN];
  mt[0] = seed;
  for (int i = 1; i < NN; ++i)
    mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) +
            (uint64_t)i;
  int idx = NN;
  for (int64_t k = 0; k < n; ++k) {
    if (idx >= NN) {
      for (int i = 0; i < NN; ++i) {
        const uint64_t x = (mt[i] & UM) | (mt[(i + 1) % NN] & LM);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= A;
        mt[i] = mt[(i + MM) % NN] ^ xa;
      }
      idx = 0;
    }
    uint64_t y = mt[idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    double u = (double)y / 18446744073709551616.0;
    if (u >= 1.0) u = nextafter(1.0, 0.0);
    out[k] = u * (1.0 - -1.0) + -1.0;
  }
}

static double norm2(const double* v, int64_t n) { /* spectral.cpp:10-14 */
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
  return sqrt(s);
}

/* estimate_spectral_radius — P/src/spectral.cpp:26-71 */
int oc_estimate_rho_cb(oc_rhs_fn f, void* ctx, int64_t n, double t,
                       const double* y, const double* v0, double rho0,
                       emrkc_rho_result* out, double* v_out) {
  const double kEps = 1e-8, kTol = 1e-2;
  const int kMaxIters = 50;
  double* v = (double*)malloc(sizeof(double) * n);
  double* fy = (double*)malloc(sizeof(double) * n);
  double* fz = (double*)malloc(sizeof(double) * n);
  double* z = (double*)malloc(sizeof(double) * n);
  int rc = 0;
  if (!v || !fy || !fz || !z) {
    rc = fail(EMRKC_ENOMEM, "out of memory");
    goto done;
  }
  if (v0)
    memcpy(v, v0, sizeof(double) * n);
  else
    oc_mt19937_64_uniform(0x9e3779b97f4a7c15ULL, n, v);
  out->safety = 1.05;
  out->converged = 1;
  if (norm2(v, n) == 0.0) {
    rc = fail(EMRKC_EINVAL, "estimate_spectral_radius: v0 must be nonzero");
    goto done;
  }
  const double ny = norm2(y, n);
  const double delta = (ny > kEps ? ny : kEps) * kEps;
  f(ctx, t, y, fy, n);
  double rho = rho0, rho_old = 0.0;
  int it = 0;
  while (it == 0 || fabs(rho - rho_old) >= kTol * rho) {
    if (it >= kMaxIters) {
      out->converged = 0;
      break;
    }
    rho_old = rho;
    const double q = delta / norm2(v, n);
    for (int64_t i = 0; i < n; ++i) z[i] = y[i] + q * v[i];
    f(ctx, t, z, fz, n);
    for (int64_t i = 0; i < n; ++i) v[i] = fz[i] - fy[i];
    const double nv = norm2(v, n);
    if (nv < 1e-300) {
      out->rho = 0.0;
      out->iterations = it + 1;
      goto vout;
    }
    rho = nv / delta;
    ++it;
  }
  out->rho = rho * out->safety;
  out->iterations = it;
vout:
  if (v_out) memcpy(v_out, v, sizeof(double) * n);
done:
  free(v);
  free(fy);
  free(fz);
  free(z);
  return rc;
}

typedef struct grid_ctx {
  const emrkc_problem* p;
  int32_t stiff; /* gate mask of the fast part (mRKC stiff-gate split) */
} grid_ctx;

/* gate_rows — P/src/monodomain.cpp:223-236: out[g] = Lambda_g (z_g - z_inf_g)
 * for the gates in mask */
static void gate_rows(const emrkc_problem* p, const double* y, double* out, int32_t mask) {
  const int64_t nn = n_nodes(p);
  if (!(mask & 7)) return;
  for (int64_t i = 0; i < nn; ++i) {
    double lam[3], zi[3];
    oc_hh_gate_coeffs(y[i], lam, zi);
    for (int g = 0; g < 3; ++g)
      if (mask >> g & 1) {
        const int64_t k = (1 + g) * nn + i;
        out[k] = lam[g] * (y[k] - zi[g]);
      }
  }
}

/* f_F_with_gates / f_S_with_gates — P/src/monodomain.cpp:287-304 */
void oc_f_F_gates(const emrkc_problem* p, int32_t stiff, double t, const double* y,
                  double* out) {
  oc_f_F(p, t, y, out);
  gate_rows(p, y, out, stiff);
}
void oc_f_S_gates(const emrkc_problem* p, int32_t stiff, double t, const double* y,
                  double* out) {
  oc_f_S(p, t, y, out);
  gate_rows(p, y, out, ~stiff & 7);
}

static void grid_fF(void* c, double t, const double* y, double* out,
                    int64_t n) {
  (void)n;
  oc_f_F(((grid_ctx*)c)->p, t, y, out);
}
static void grid_fS(void* c, double t, const double* y, double* out,
                    int64_t n) {
  (void)n;
  oc_f_S(((grid_ctx*)c)->p, t, y, out);
}
static void grid_fFg(void* c, double t, const double* y, double* out, int64_t n) {
  (void)n;
  oc_f_F_gates(((grid_ctx*)c)->p, ((grid_ctx*)c)->stiff, t, y, out);
}
static void grid_fSg(void* c, double t, const double* y, double* out, int64_t n) {
  (void)n;
  oc_f_S_gates(((grid_ctx*)c)->p, ((grid_ctx*)c)->stiff, t, y, out);
}
static void grid_exp(void* c, const double* y, double* lam, double* yinf,
                     int64_t n) {
  (void)n;
  oc_exp_part(((grid_ctx*)c)->p, y, lam, yinf);
}

int oc_estimate_rho(const emrkc_problem* p, int32_t which, double t,
                    const double* y, const double* v0, double rho0,
                    emrkc_rho_result* out, double* v_out) {
  int rc = oc_validate(p);
  if (rc) return rc;
  /* which: EMRKC_RHS_F / _S, or 2 / 3 = f_F / f_S with gate rows, stiff
   * gate mask in bits 4.. (mRKC split) */
  grid_ctx c = {p, (which >> 4) & 7};
  oc_rhs_fn f = grid_fF;
  switch (which & 15) {
    case EMRKC_RHS_F: f = grid_fF; break;
    case EMRKC_RHS_S: f = grid_fS; break;
    case 2: f = grid_fFg; break;
    case 3: f = grid_fSg; break;
    default: return fail(EMRKC_EINVAL, "estimate_rho: unknown rhs");
  }
  return oc_estimate_rho_cb(f, &c, oc_state_len(p), t, y, v0, rho0, out, v_out);
}

/* identify_stiff_gates — P/src/ionic.cpp:130-146: gates ordered by the
 * largest alpha + beta over the V samples, descending (stable) */
int oc_identify_stiff_gates(const double* V, int64_t n, int32_t* order) {
  if (n < 1) return fail(EMRKC_EINVAL, "identify_stiff_gates: empty trajectory");
  double mr[3] = {0.0, 0.0, 0.0};
  for (int64_t i = 0; i < n; ++i) {
    double a[3], b[3];
    oc_hh_rates(V[i], a, b);
    for (int g = 0; g < 3; ++g) {
      const double r = a[g] + b[g];
      mr[g] = (mr[g] < r) ? r : mr[g]; /* std::max */
    }
  }
  int32_t o[3] = {0, 1, 2};
  for (int i = 1; i < 3; ++i) /* stable insertion sort, descending */
    for (int j = i; j > 0 && mr[o[j - 1]] < mr[o[j]]; --j) {
      const int32_t tmp = o[j];
      o[j] = o[j - 1];
      o[j - 1] = tmp;
    }
  for (int g = 0; g < 3; ++g) order[g] = o[g];
  return 0;
}

/* ======================= run loop (P/src/simulate.cpp) ================== */

int oc_emrkc_step_grid(const emrkc_problem* p, double t, const double* y,
                       double dt, double eps, double rho_F, double rho_S,
                       double* out, emrkc_step_report* rep) {
  int rc = oc_validate(p);
  if (rc) return rc;
  grid_ctx c = {p, 0};
  oc_counters ctr = {0, 0, 0};
  oc_split rhs = {grid_fF, grid_fS, grid_exp, &c, rho_F, rho_S, &ctr};
  return oc_emrkc_step(t, y, oc_state_len(p), dt, &rhs, eps, out, rep);
}

/* track_gate_range — P/src/simulate.cpp:76-85 (std::min / std::max) */
static void track_gate_range(const double* y, int64_t nn, int64_t len,
                             double* lo, double* hi) {
  for (int64_t k = nn; k < len; ++k) {
    *lo = (y[k] < *lo) ? y[k] : *lo;
    *hi = (*hi < y[k]) ? y[k] : *hi;
  }
}

int oc_run(const emrkc_problem* p, double* y, int64_t step0, int64_t nsteps,
           double dt, double eps, double rho_F, double rho_S,
           emrkc_run_result* res, double* wall_s) {
  return oc_run_method(p, y, step0, nsteps, dt, eps, OC_METHOD_EMRKC, rho_F, rho_S, res,
                       wall_s);
}

/* rush_larsen_update + exex_rl_step — P/src/baselines.cpp:89-128,192-210
 * (HH: no auxiliary variables) */
int oc_exex_rl_step(const emrkc_problem* p, double t, const double* y, double dt,
                    double* out) {
  if (!(dt > 0.0)) return fail(EMRKC_EINVAL, "exex_rl_step: dt must be > 0");
  const int64_t nn = n_nodes(p);
  double* dv = (double*)malloc(sizeof(double) * nn);
  if (!dv) return fail(EMRKC_ENOMEM, "out of memory");
  memcpy(out, y, sizeof(double) * 4 * nn); /* ynew = y */
  for (int64_t i = 0; i < nn; ++i) { /* gate_coeffs_field on y; expm1 update */
    double lam[3], zinf[3];
    oc_hh_gate_coeffs(y[i], lam, zinf);
    for (int g = 0; g < 3; ++g) {
      const int64_t idx = (1 + g) * nn + i;
      out[idx] = y[idx] + expm1(dt * lam[g]) * (y[idx] - zinf[g]);
    }
  }
  /* v_rhs = v_reaction(t, ynew): V old, gates new; dv = diffusion(V old) */
  oc_diffusion_apply(p, y, dv);
  for (int64_t i = 0; i < nn; ++i) {
    const double z[3] = {out[nn + i], out[2 * nn + i], out[3 * nn + i]};
    const double v_rhs = oc_stimulus_rate(p, t, i) - oc_hh_ionic_current(y[i], z) / p->C_m;
    out[i] = y[i] + dt * (dv[i] + v_rhs);
  }
  free(dv);
  return 0;
}

/* cg_solve — P/src/baselines.cpp:20-82 on the IMEX operator
 * op(u) = u - dt sqrt(w) D(u / sqrt(w)) (:150-158) */
static double dotv(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

typedef struct imex_op {
  const emrkc_problem* p;
  const double* sw;
  const double* isw;
  double dt;
  double* unscaled;
  double* scratch;
} imex_op;

static void imex_apply(const imex_op* o, const double* u, double* out, int64_t nn) {
  for (int64_t i = 0; i < nn; ++i) o->unscaled[i] = o->isw[i] * u[i];
  oc_diffusion_apply(o->p, o->unscaled, o->scratch);
  for (int64_t i = 0; i < nn; ++i) out[i] = u[i] - o->dt * o->sw[i] * o->scratch[i];
}

/* quadrature_weights — P/src/monodomain.cpp:52-63 */
static void quad_weights(const emrkc_problem* p, double* w) {
  const int64_t nn = n_nodes(p);
  for (int64_t i = 0; i < nn; ++i) w[i] = 1.0;
  for (int a = 0; a < p->dim; ++a) {
    const int64_t stride = axis_stride(p, a), na = p->n[a];
    for (int64_t i = 0; i < nn; ++i) {
      const int64_t ia = (i / stride) % na;
      if (ia == 0 || ia == na - 1) w[i] *= 0.5;
    }
  }
}

/* imex_rl_step — P/src/baselines.cpp:132-190 (HH). Returns EMRKC_ENONFINITE
 * when CG does not converge; *iters = CG iterations, *applies = op applies. */
int oc_imex_rl_step(const emrkc_problem* p, double t, const double* y, double dt,
                    double rel_tol, int64_t max_iters, int32_t jacobi, double* out,
                    int64_t* iters, int64_t* applies) {
  if (!(dt > 0.0)) return fail(EMRKC_EINVAL, "imex_rl_step: dt must be > 0");
  const int64_t nn = n_nodes(p);
  double* buf = (double*)malloc(sizeof(double) * 13 * nn);
  if (!buf) return fail(EMRKC_ENOMEM, "out of memory");
  double *w = buf, *sw = buf + nn, *isw = buf + 2 * nn, *un = buf + 3 * nn, *sc = buf + 4 * nn;
  double *b = buf + 5 * nn, *x = buf + 6 * nn, *r = buf + 7 * nn, *z = buf + 8 * nn;
  double *pp = buf + 9 * nn, *q = buf + 10 * nn, *vr = buf + 11 * nn, *e = buf + 12 * nn;
  /* rush_larsen_update (:89-128): gates at y's V, reaction at the new gates */
  memcpy(out, y, sizeof(double) * 4 * nn);
  for (int64_t i = 0; i < nn; ++i) {
    double lam[3], zinf[3];
    oc_hh_gate_coeffs(y[i], lam, zinf);
    for (int g = 0; g < 3; ++g) {
      const int64_t idx = (1 + g) * nn + i;
      out[idx] = y[idx] + expm1(dt * lam[g]) * (y[idx] - zinf[g]);
    }
  }
  for (int64_t i = 0; i < nn; ++i) {
    const double zz[3] = {out[nn + i], out[2 * nn + i], out[3 * nn + i]};
    vr[i] = oc_stimulus_rate(p, t, i) - oc_hh_ionic_current(y[i], zz) / p->C_m;
  }
  quad_weights(p, w);
  for (int64_t i = 0; i < nn; ++i) {
    sw[i] = sqrt(w[i]);
    isw[i] = 1.0 / sw[i];
  }
  imex_op o = {p, sw, isw, dt, un, sc};
  for (int64_t i = 0; i < nn; ++i) {
    b[i] = sw[i] * (y[i] + dt * vr[i]);
    x[i] = sw[i] * y[i];
  }
  for (int64_t i = 0; i < nn; ++i) e[i] = 0.0;
  e[0] = 1.0;
  oc_diffusion_apply(p, e, sc);
  const double diag = 1.0 - dt * sc[0];
  /* cg_solve */
  int64_t it = 0, ap = 0;
  int converged = 1;
  const double nb = sqrt(dotv(b, b, nn));
  if (nb == 0.0) {
    for (int64_t i = 0; i < nn; ++i) x[i] = 0.0;
  } else {
    const int64_t max_it =
        max_iters > 0 ? max_iters : (int64_t)(10.0 * sqrt((double)nn)) + 1;
    imex_apply(&o, x, q, nn);
    ++ap;
    for (int64_t i = 0; i < nn; ++i) r[i] = b[i] - q[i];
    for (int64_t i = 0; i < nn; ++i) z[i] = jacobi ? r[i] / diag : r[i];
    memcpy(pp, z, sizeof(double) * nn);
    double rz = dotv(r, z, nn);
    double rnorm = sqrt(dotv(r, r, nn));
    const double tol = rel_tol * nb;
    while (rnorm > tol) {
      if (it >= max_it) {
        converged = 0;
        break;
      }
      imex_apply(&o, pp, q, nn);
      ++ap;
      const double alpha = rz / dotv(pp, q, nn);
      for (int64_t i = 0; i < nn; ++i) {
        x[i] += alpha * pp[i];
        r[i] -= alpha * q[i];
      }
      for (int64_t i = 0; i < nn; ++i) z[i] = jacobi ? r[i] / diag : r[i];
      const double rz_new = dotv(r, z, nn);
      const double beta = rz_new / rz;
      rz = rz_new;
      for (int64_t i = 0; i < nn; ++i) pp[i] = z[i] + beta * pp[i];
      rnorm = sqrt(dotv(r, r, nn));
      ++it;
    }
  }
  *iters = it;
  *applies = ap;
  int rc = 0;
  if (!converged)
    rc = fail(EMRKC_ENONFINITE, "imex_rl_step: CG did not converge");
  else
    for (int64_t i = 0; i < nn; ++i) out[i] = isw[i] * x[i];
  free(buf);
  return rc;
}

/* run_simulation's imex_rl loop (P/src/simulate.cpp:176-229) */
int oc_run_imex(const emrkc_problem* p, double* y, int64_t step0, int64_t nsteps, double dt,
                double rel_tol, int64_t max_iters, int32_t jacobi, emrkc_run_result* res,
                int64_t* cg_iters_total) {
  int rc = oc_validate(p);
  if (rc) return rc;
  if (n_aux_of(p)) return fail(EMRKC_EINVAL, "hh_aux: emRKC (standard / progressive) only");
  const int64_t nn = n_nodes(p), len = 4 * nn;
  double* next = (double*)malloc(sizeof(double) * len);
  if (!next) return fail(EMRKC_ENOMEM, "out of memory");
  memset(res, 0, sizeof(*res));
  res->n_steps = nsteps;
  res->abort_step = -1;
  res->gate_min = 1.0;
  res->gate_max = 0.0;
  res->s = res->m = 1;
  res->eta = dt;
  track_gate_range(y, nn, 4 * nn, &res->gate_min, &res->gate_max);
  int64_t tot = 0;
  for (int64_t step = step0; step < step0 + nsteps; ++step) {
    const double t = (double)step * dt;
    int64_t it = 0, ap = 0;
    rc = oc_imex_rl_step(p, t, y, dt, rel_tol, max_iters, jacobi, next, &it, &ap);
    ++res->n_exp; /* rush_larsen_update (:105-106,123-124) */
    ++res->n_fS;
    res->n_fF += ap + 1; /* probe + solve applies (:181) */
    tot += it;
    if (rc == EMRKC_ENONFINITE) {
      res->aborted = 1;
      res->abort_kind = EMRKC_ABORT_NONFINITE;
      res->abort_step = step;
      res->abort_stage = -1;
      rc = 0;
      break;
    }
    if (rc) break;
    memcpy(y, next, sizeof(double) * len);
    ++res->steps_done;
    double mv = 0.0;
    for (int64_t i = 0; i < nn; ++i) {
      if (!isfinite(y[i])) {
        mv = INFINITY;
        break;
      }
      const double ay = fabs(y[i]);
      mv = (mv < ay) ? ay : mv;
    }
    if (mv > 1e6) {
      res->aborted = 1;
      res->abort_kind = EMRKC_ABORT_NORM_GUARD;
      res->abort_step = step;
      break;
    }
    track_gate_range(y, nn, 4 * nn, &res->gate_min, &res->gate_max);
  }
  if (cg_iters_total) *cg_iters_total = tot;
  free(next);
  return rc;
}

/* run_simulation's stepping loop — P/src/simulate.cpp:110-113, 176-229:
 * the emRKC / emRKC-progressive branches (:197-207) and exex_rl (:211-212) */
int oc_run_mrkc(const emrkc_problem* p, double* y, int64_t step0, int64_t nsteps,
                double dt, double eps, int32_t stiff, double rho_F, double rho_S,
                emrkc_run_result* res, double* wall_s) {
  return oc_run_method(p, y, step0, nsteps, dt, eps, OC_METHOD_MRKC | ((stiff & 7) << 4), rho_F,
                       rho_S, res, wall_s);
}

int oc_run_method(const emrkc_problem* p, double* y, int64_t step0, int64_t nsteps,
                  double dt, double eps, int32_t method, double rho_F, double rho_S,
                  emrkc_run_result* res, double* wall_s) {
  const int32_t stiff = (method >> 4) & 7;
  method &= 15;
  int rc = oc_validate(p);
  if (rc) return rc;
  const int64_t nn = n_nodes(p), len = oc_state_len(p);
  if (n_aux_of(p) && method != OC_METHOD_EMRKC && method != OC_METHOD_EMRKC_PROGRESSIVE)
    return fail(EMRKC_EINVAL, "hh_aux: emRKC (standard / progressive) only");
  grid_ctx c = {p, stiff};
  oc_counters ctr = {0, 0, 0};
  oc_split rhs = {grid_fF, grid_fS, grid_exp, &c, rho_F, rho_S, &ctr};
  if (method == OC_METHOD_MRKC) { /* simulate.cpp:132-150 */
    rhs.f_F = grid_fFg;
    rhs.f_S = grid_fSg;
    rhs.exp_part = NULL;
  }
  double* next = (double*)malloc(sizeof(double) * len);
  if (!next) return fail(EMRKC_ENOMEM, "out of memory");
  memset(res, 0, sizeof(*res));
  res->n_steps = nsteps;
  res->abort_step = -1;
  res->gate_min = 1.0;
  res->gate_max = 0.0;
  track_gate_range(y, nn, 4 * nn, &res->gate_min, &res->gate_max);
  struct timespec w0, w1;
  clock_gettime(CLOCK_MONOTONIC, &w0);
  for (int64_t step = step0; step < step0 + nsteps; ++step) {
    const double t = (double)step * dt;
    emrkc_step_report rep;
    if (method == OC_METHOD_EXEX_RL) {
      rc = oc_exex_rl_step(p, t, y, dt, next);
      /* counters: one exp step, one f_S, one f_F (baselines.cpp:105,123,203) */
      ++ctr.n_exp;
      ++ctr.n_fS;
      ++ctr.n_fF;
      memset(&rep, 0, sizeof rep);
      rep.s = rep.m = 1;
      rep.eta = dt;
    } else {
      rc = oc_emrkc_step_v(t, y, len, dt, &rhs, eps,
                           method == OC_METHOD_EMRKC_PROGRESSIVE ? EMRKC_VARIANT_PROGRESSIVE
                           : method == OC_METHOD_MRKC           ? OC_VARIANT_MRKC
                                                                 : EMRKC_VARIANT_STANDARD,
                           next, &rep);
    }
    if (rc == EMRKC_ENONFINITE) {
      res->aborted = 1;
      res->abort_kind = EMRKC_ABORT_NONFINITE;
      res->abort_step = step;
      res->abort_stage = rep.abort_stage;
      res->abort_inner = rep.abort_inner;
      res->abort_outer_stage = rep.abort_outer_stage;
      rc = 0;
      break;
    }
    if (rc) break;
    res->s = rep.s;
    res->m = rep.m;
    res->eta = rep.eta;
    memcpy(y, next, sizeof(double) * len);
    ++res->steps_done;
    /* max_abs_v :67-74 and the norm guard :222-227 */
    double mv = 0.0;
    for (int64_t i = 0; i < nn; ++i) {
      if (!isfinite(y[i])) {
        mv = INFINITY;
        break;
      }
      const double ay = fabs(y[i]);
      mv = (mv < ay) ? ay : mv; /* std::max */
    }
    if (mv > 1e6) {
      res->aborted = 1;
      res->abort_kind = EMRKC_ABORT_NORM_GUARD;
      res->abort_step = step;
      break;
    }
    track_gate_range(y, nn, 4 * nn, &res->gate_min, &res->gate_max);
  }
  clock_gettime(CLOCK_MONOTONIC, &w1);
  if (wall_s)
    *wall_s = (double)(w1.tv_sec - w0.tv_sec) + 1e-9 * (w1.tv_nsec - w0.tv_nsec);
  res->n_fF = ctr.n_fF;
  res->n_fS = ctr.n_fS;
  res->n_exp = ctr.n_exp;
  free(next);
  return rc;
}

/* ============ scalar surrogates (P/tests/test_multirate.cpp:54-66) ========= */

typedef struct scalar_ctx {
  double lF, lS, lE, yinf;
} scalar_ctx;

static void sc_fF(void* c, double t, const double* y, double* out, int64_t n) {
  (void)t;
  (void)n;
  out[0] = ((scalar_ctx*)c)->lF * y[0];
}
static void sc_fS(void* c, double t, const double* y, double* out, int64_t n) {
  (void)t;
  (void)n;
  out[0] = ((scalar_ctx*)c)->lS * y[0];
}
static void sc_exp(void* c, const double* y, double* lam, double* yinf,
                   int64_t n) {
  (void)y;
  (void)n;
  lam[0] = ((scalar_ctx*)c)->lE;
  yinf[0] = ((scalar_ctx*)c)->yinf;
}

int oc_scalar_averaged_force(double lF, double lS, double lE, double yinf,
                             double y, double eta, int32_t m, double eps,
                             double* out) {
  scalar_ctx c = {lF, lS, lE, yinf};
  oc_split rhs = {sc_fF, sc_fS, sc_exp, &c, fabs(lF), fabs(lS), NULL};
  int32_t st = 0;
  return oc_averaged_force_emrkc(0.0, &y, 1, eta, &rhs, m, eps, out, &st);
}

int oc_scalar_emrkc_step(double lF, double lS, double lE, double yinf,
                         double y, double dt, double eps, double* out,
                         int32_t* s, int32_t* m, double* eta) {
  scalar_ctx c = {lF, lS, lE, yinf};
  oc_split rhs = {sc_fF, sc_fS, sc_exp, &c, fabs(lF), fabs(lS), NULL};
  emrkc_step_report rep;
  const int rc = oc_emrkc_step(0.0, &y, 1, dt, &rhs, eps, out, &rep);
  *s = rep.s;
  *m = rep.m;
  *eta = rep.eta;
  return rc;
}
