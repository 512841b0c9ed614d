// emrkc_generic.cu — the reference's integrator layer over device callbacks
// (include/emrkc.h "integrator layer"): rkc_iteration, exponential Euler,
// the emRKC / mRKC averaged forces and steps, and the nonlinear power
// iteration, for any SplitRhs whose callbacks enqueue their work on a CUDA
// stream. P/ = /root/reference/proj.
//
// The arithmetic follows the reference operation for operation (explicit
// _rn intrinsics: no FMA contraction, as in the reference's x86-64 build):
//   stage 1  g1 = y + (mu_1 dt) f                      P/src/cheb.cpp:91
//   stage j  g_j = (nu_j g_{j-1} + kappa_j g_{j-2}) + (mu_j dt) f   :98-99
//   expEuler y + expm1(eta L) (y - y_inf)              P/src/multirate.cpp:56
//   f_u      f_F(u) + fs   |  f_F(u) + (fs + expc)      :101-102, :111-112
//   force    (u - y) / eta                              :117
//   power    z = y + q v,  v = f(z) - f(y)              P/src/spectral.cpp:57-59
// Norms are summed in the reference's serial order (bit-identical). Finite
// checks are device flags read once per stage, so NumericalAbort names the
// same stage and the
// callback counts match the reference's exactly. This is not the hot path:
// the fused emrkc_step kernels (kernels_fast.cu) are; this layer makes the
// reference's generic API (and its scalar known-answer tests) run on the
// device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "../../include/emrkc.h"
#include "kernels.h"

struct emrkc_vctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int* d_flag = nullptr;     // non-finite flag of a stage
  int* h_flag = nullptr;     // pinned
  double* d_part = nullptr;  // reduction partials [kRedBlocks] + result
  double* h_sum = nullptr;   // pinned
};

namespace {

constexpr int kThreads = 256;
constexpr int kRedBlocks = 296;  // 2 x 148 SMs

int fail(emrkc_vctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define GK(c, call)                                                             \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess)                                                      \
      return fail((c), EMRKC_ECUDA, "%s: %s", #call, cudaGetErrorString(e_));   \
  } while (0)

int grid_for(int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads,
                                                                  148 * 16)));
}

__global__ void k_stage1(double* __restrict__ out, const double* __restrict__ y, double c,
                         const double* __restrict__ f, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __dadd_rn(y[i], __dmul_rn(c, f[i]));
}

// gm2 <- nu gm1 + kappa gm2 + (mu dt) f (P/src/cheb.cpp:98-99)
__global__ void k_stagej(double* __restrict__ gm2, const double* __restrict__ gm1, double nu,
                         double kappa, double c, const double* __restrict__ f, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    gm2[i] = __dadd_rn(__dadd_rn(__dmul_rn(nu, gm1[i]), __dmul_rn(kappa, gm2[i])),
                       __dmul_rn(c, f[i]));
}

__global__ void k_nonfinite(const double* __restrict__ x, int64_t n, int* flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

__global__ void k_expeuler(double* out, const double* y, double eta, const double* __restrict__ lam,
                           const double* __restrict__ yinf, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double yi = y[i];
    out[i] = __dadd_rn(yi, __dmul_rn(expm1(__dmul_rn(eta, lam[i])), __dsub_rn(yi, yinf[i])));
  }
}

// out += a  |  out += (a + b)
__global__ void k_add(double* __restrict__ out, const double* __restrict__ a,
                      const double* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __dadd_rn(out[i], b ? __dadd_rn(a[i], b[i]) : a[i]);
}

// out = (u - y) / eta
__global__ void k_diffdiv(double* out, const double* u, const double* __restrict__ y, double eta,
                          int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __ddiv_rn(__dsub_rn(u[i], y[i]), eta);
}

// z = y + q v
__global__ void k_zaxpy(double* __restrict__ z, const double* __restrict__ y, double q,
                        const double* __restrict__ v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    z[i] = __dadd_rn(y[i], __dmul_rn(q, v[i]));
}

// v = a - b
__global__ void k_sub(double* __restrict__ v, const double* __restrict__ a,
                      const double* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = __dsub_rn(a[i], b[i]);
}

// Device scratch, released on scope exit (stream-ordered).
struct Scratch {
  emrkc_vctx* c;
  std::vector<double*> bufs;
  explicit Scratch(emrkc_vctx* c_) : c(c_) {}
  ~Scratch() {
    for (double* p : bufs) cudaFreeAsync(p, c->stream);
  }
  double* get(int64_t n) {
    double* p = nullptr;
    if (cudaMallocAsync(&p, sizeof(double) * std::max<int64_t>(n, 1), c->stream) != cudaSuccess)
      return nullptr;
    bufs.push_back(p);
    return p;
  }
};

int use(emrkc_vctx* c) {
  GK(c, cudaSetDevice(c->device));
  return EMRKC_OK;
}

int stage_nonfinite(emrkc_vctx* c, const double* x, int64_t n, bool* bad) {
  GK(c, cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
  k_nonfinite<<<grid_for(n), kThreads, 0, c->stream>>>(x, n, c->d_flag);
  GK(c, cudaGetLastError());
  GK(c, cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  GK(c, cudaStreamSynchronize(c->stream));
  *bad = *c->h_flag != 0;
  return EMRKC_OK;
}

// ||x|| in the reference's serial order (P/src/spectral.cpp:10-14),
// bit-identical to it (kernels.cu k_sumsq_serial).
int norm2(emrkc_vctx* c, const double* x, int64_t n, double* out) {
  GK(c, emrkc_k::launch_sumsq_serial(x, n, 0.0, c->d_part + kRedBlocks, c->stream));
  GK(c, cudaMemcpyAsync(c->h_sum, c->d_part + kRedBlocks, sizeof(double),
                        cudaMemcpyDeviceToHost, c->stream));
  GK(c, cudaStreamSynchronize(c->stream));
  *out = std::sqrt(*c->h_sum);
  return EMRKC_OK;
}

// A right-hand side as the iteration sees it: a callback, or the averaged
// force of the outer iteration (recursion through this closure).
struct Rhs {
  virtual int eval(double t, const double* y, double* out, int64_t n, int32_t* inner_bad) = 0;
  virtual ~Rhs() = default;
};

struct CallbackRhs : Rhs {
  emrkc_vctx* c;
  emrkc_rhs_fn f;
  void* ctx;
  int64_t* counter;
  const double* add_a = nullptr;  // f_u = f(u) + a (+ b)
  const double* add_b = nullptr;
  int eval(double t, const double* y, double* out, int64_t n, int32_t*) override {
    if (f(ctx, t, y, out, n, c->stream)) return fail(c, EMRKC_ECALLBACK, "rhs callback failed");
    if (counter) ++*counter;
    if (add_a) {
      k_add<<<grid_for(n), kThreads, 0, c->stream>>>(out, add_a, add_b, n);
      GK(c, cudaGetLastError());
    }
    return EMRKC_OK;
  }
};

// rkc_iteration (P/src/cheb.cpp:84-105) with coefficients for (s, eps).
int rkc_iter(emrkc_vctx* c, double t, const double* y, int64_t n, double dt, Rhs& f, int s,
             double eps, double* out, int32_t* bad_stage, int32_t* inner_bad) {
  if (s < 1) return fail(c, EMRKC_EINVAL, "rkc_coeffs: s must be >= 1");
  std::vector<double> b(s + 1), mu(s + 1), nu(s + 1), ka(s + 1), cc(s + 1);
  double w0 = 0, w1 = 0;
  int rc = emrkc_rkc_coeffs(s, eps, &w0, &w1, b.data(), mu.data(), nu.data(), ka.data(),
                            cc.data());
  if (rc) return fail(c, rc, "%s", emrkc_global_error());
  Scratch sc(c);
  double* fbuf = sc.get(n);
  double* gA = sc.get(n);  // g_{j-1}
  double* gB = sc.get(n);  // g_{j-2}
  if (!fbuf || !gA || !gB) return fail(c, EMRKC_ENOMEM, "rkc_iteration: out of device memory");
  if ((rc = f.eval(t, y, fbuf, n, inner_bad))) return rc;
  GK(c, cudaMemcpyAsync(gB, y, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  k_stage1<<<grid_for(n), kThreads, 0, c->stream>>>(gA, y, mu[1] * dt, fbuf, n);
  GK(c, cudaGetLastError());
  bool bad = false;
  if ((rc = stage_nonfinite(c, gA, n, &bad))) return rc;
  if (bad) {
    if (bad_stage) *bad_stage = 1;
    return fail(c, EMRKC_ENONFINITE, "rkc_iteration: non-finite value at stage 1");
  }
  for (int j = 2; j <= s; ++j) {
    if ((rc = f.eval(t + cc[j - 1] * dt, gA, fbuf, n, inner_bad))) return rc;
    k_stagej<<<grid_for(n), kThreads, 0, c->stream>>>(gB, gA, nu[j], ka[j], mu[j] * dt, fbuf, n);
    GK(c, cudaGetLastError());
    std::swap(gA, gB);
    if ((rc = stage_nonfinite(c, gA, n, &bad))) return rc;
    if (bad) {
      if (bad_stage) *bad_stage = j;
      return fail(c, EMRKC_ENONFINITE, "rkc_iteration: non-finite value at stage %d", j);
    }
  }
  GK(c, cudaMemcpyAsync(out, gA, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  return EMRKC_OK;
}

// averaged_force_emrkc / _mrkc (P/src/multirate.cpp:60-119). variant:
// 0 standard, 1 progressive, 2 mRKC.
int averaged(emrkc_vctx* c, double t, const double* y, int64_t n, double eta,
             const emrkc_split_rhs* rhs, int m, int variant, double eps, double* out,
             int32_t* bad_stage) {
  if (m < 1)
    return fail(c, EMRKC_EINVAL, variant == 2 ? "averaged_force_mrkc: m must be >= 1"
                                              : "averaged_force_emrkc: m must be >= 1");
  if (!rhs || !rhs->f_F || !rhs->f_S) return fail(c, EMRKC_EINVAL, "SplitRhs: f_F / f_S missing");
  if (variant != 2 && !rhs->exp_part)
    return fail(c, EMRKC_EINVAL, "averaged_force_emrkc: exp_part missing");
  Scratch sc(c);
  double* fs = sc.get(n);
  double* u = sc.get(n);
  if (!fs || !u) return fail(c, EMRKC_ENOMEM, "averaged force: out of device memory");
  emrkc_counters* ctr = rhs->counters;
  CallbackRhs fu;
  fu.c = c;
  fu.f = rhs->f_F;
  fu.ctx = rhs->f_F_ctx;
  fu.counter = ctr ? &ctr->n_fF : nullptr;
  fu.add_a = fs;
  int rc;
  const double* start = y;
  if (variant == 2) {
    if (rhs->f_S(rhs->f_S_ctx, t, y, fs, n, c->stream))
      return fail(c, EMRKC_ECALLBACK, "f_S callback failed");
    if (ctr) ++ctr->n_fS;
  } else {
    double* lam = sc.get(n);
    double* yinf = sc.get(n);
    double* yE = sc.get(n);
    if (!lam || !yinf || !yE) return fail(c, EMRKC_ENOMEM, "averaged force: out of device memory");
    if (rhs->exp_part(rhs->exp_ctx, y, lam, yinf, n, c->stream))
      return fail(c, EMRKC_ECALLBACK, "exp_part callback failed");
    k_expeuler<<<grid_for(n), kThreads, 0, c->stream>>>(yE, y, eta, lam, yinf, n);
    GK(c, cudaGetLastError());
    if (ctr) ++ctr->n_exp_steps;
    if (rhs->f_S(rhs->f_S_ctx, t, yE, fs, n, c->stream))
      return fail(c, EMRKC_ECALLBACK, "f_S callback failed");
    if (ctr) ++ctr->n_fS;
    if (variant == 0) {
      start = yE;
    } else {
      // expc = (y_E - y) / eta, then f_u = f_F(u) + (fs + expc)
      k_diffdiv<<<grid_for(n), kThreads, 0, c->stream>>>(lam, yE, y, eta, n);
      GK(c, cudaGetLastError());
      fu.add_b = lam;
    }
  }
  int32_t dummy = 0;
  if ((rc = rkc_iter(c, t, start, n, eta, fu, m, eps, u, bad_stage, &dummy))) return rc;
  k_diffdiv<<<grid_for(n), kThreads, 0, c->stream>>>(out, u, y, eta, n);
  GK(c, cudaGetLastError());
  return EMRKC_OK;
}

struct AveragedRhs : Rhs {
  emrkc_vctx* c;
  const emrkc_split_rhs* rhs;
  double eta, eps;
  int m, variant;
  int32_t inner_stage = 0;
  int eval(double t, const double* y, double* out, int64_t n, int32_t* inner_bad) override {
    int32_t st = 0;
    const int rc = averaged(c, t, y, n, eta, rhs, m, variant, eps, out, &st);
    if (rc == EMRKC_ENONFINITE) {
      inner_stage = st;
      if (inner_bad) *inner_bad = 1;
    }
    return rc;
  }
};

int step_split(emrkc_vctx* c, double t, const double* y, int64_t n, double dt,
               const emrkc_split_rhs* rhs, double eps, int variant, double* out,
               emrkc_step_report* rep) {
  const char* name = variant == 2 ? "mrkc_step" : "emrkc_step";
  if (!(dt > 0.0)) return fail(c, EMRKC_EINVAL, "%s: dt must be > 0", name);
  if (!rhs) return fail(c, EMRKC_EINVAL, "null SplitRhs");
  if (variant != 2 && !rhs->exp_part) return fail(c, EMRKC_EINVAL, "emrkc_step: exp_part missing");
  // plan_step (P/src/multirate.cpp:129-135)
  int32_t s = 0, m = 0;
  double ell_s = 0, ell_m = 0, beta = 0;
  int rc = emrkc_get_stages(dt, rhs->rho_S, eps, &s, &ell_s, &beta);
  if (rc) return fail(c, rc, "%s", emrkc_global_error());
  const double eta = 2.0 * dt / ell_s;
  if ((rc = emrkc_get_stages(eta, rhs->rho_F, eps, &m, &ell_m, &beta)))
    return fail(c, rc, "%s", emrkc_global_error());
  const emrkc_counters before = rhs->counters ? *rhs->counters : emrkc_counters{};
  AveragedRhs av;
  av.c = c;
  av.rhs = rhs;
  av.eta = eta;
  av.eps = eps;
  av.m = m;
  av.variant = variant;
  int32_t bad = 0, inner = 0;
  rc = rkc_iter(c, t, y, n, dt, av, s, eps, out, &bad, &inner);
  if (rep) {
    *rep = emrkc_step_report{};
    rep->s = s;
    rep->m = m;
    rep->eta = eta;
    rep->ell_s = ell_s;
    rep->ell_m = ell_m;
    if (rhs->counters) {
      rep->n_fF = rhs->counters->n_fF - before.n_fF;
      rep->n_fS = rhs->counters->n_fS - before.n_fS;
      rep->n_exp = rhs->counters->n_exp_steps - before.n_exp_steps;
    }
    if (rc == EMRKC_ENONFINITE) {
      rep->abort_kind = EMRKC_ABORT_NONFINITE;
      rep->abort_inner = inner;
      rep->abort_stage = inner ? av.inner_stage : bad;
    }
  }
  return rc;
}

// seeded_direction (P/src/spectral.cpp:16-22): libstdc++ mt19937_64 +
// uniform_real_distribution(-1, 1) — the reference's generator itself.
std::vector<double> seeded_direction(int64_t n) {
  std::mt19937_64 rng(0x9e3779b97f4a7c15ull);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  std::vector<double> v(n);
  for (double& x : v) x = dist(rng);
  return v;
}

}  // namespace

extern "C" {

int emrkc_vctx_create(int32_t device, emrkc_vctx** out) {
  if (!out) return EMRKC_EINVAL;
  *out = nullptr;
  auto* c = new emrkc_vctx();
  c->device = device;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
    delete c;
    return EMRKC_ECUDA;  // no CPU fallback
  }
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&c->d_flag, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&c->d_part, sizeof(double) * (kRedBlocks + 1)) != cudaSuccess ||
      cudaHostAlloc(&c->h_flag, sizeof(int), 0) != cudaSuccess ||
      cudaHostAlloc(&c->h_sum, sizeof(double), 0) != cudaSuccess) {
    emrkc_vctx_destroy(c);
    return EMRKC_ECUDA;
  }
  *out = c;
  return EMRKC_OK;
}

void emrkc_vctx_destroy(emrkc_vctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  cudaFree(c->d_flag);
  cudaFree(c->d_part);
  cudaFreeHost(c->h_flag);
  cudaFreeHost(c->h_sum);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* emrkc_vctx_last_error(const emrkc_vctx* c) { return c ? c->err.c_str() : ""; }
void* emrkc_vctx_stream(emrkc_vctx* c) { return c ? (void*)c->stream : nullptr; }

int emrkc_vctx_alloc(emrkc_vctx* c, int64_t len, double** dptr) {
  if (!c || !dptr || len < 0) return EMRKC_EINVAL;
  int rc = use(c);
  if (rc) return rc;
  GK(c, cudaMallocAsync(dptr, sizeof(double) * std::max<int64_t>(len, 1), c->stream));
  GK(c, cudaStreamSynchronize(c->stream));
  return EMRKC_OK;
}
int emrkc_vctx_free(emrkc_vctx* c, double* dptr) {
  if (!c) return EMRKC_EINVAL;
  int rc = use(c);
  if (rc) return rc;
  GK(c, cudaFreeAsync(dptr, c->stream));
  return EMRKC_OK;
}
int emrkc_vctx_upload(emrkc_vctx* c, double* dst, const double* host, int64_t len) {
  if (!c || (!dst && len) || (!host && len)) return EMRKC_EINVAL;
  int rc = use(c);
  if (rc) return rc;
  GK(c, cudaMemcpyAsync(dst, host, sizeof(double) * len, cudaMemcpyHostToDevice, c->stream));
  GK(c, cudaStreamSynchronize(c->stream));
  return EMRKC_OK;
}
int emrkc_vctx_download(emrkc_vctx* c, double* host, const double* src, int64_t len) {
  if (!c || (!src && len) || (!host && len)) return EMRKC_EINVAL;
  int rc = use(c);
  if (rc) return rc;
  GK(c, cudaMemcpyAsync(host, src, sizeof(double) * len, cudaMemcpyDeviceToHost, c->stream));
  GK(c, cudaStreamSynchronize(c->stream));
  return EMRKC_OK;
}

int emrkc_exponential_euler(emrkc_vctx* c, const double* y, double eta, const double* lambda,
                            const double* y_inf, int64_t len, double* out) {
  if (!c) return EMRKC_EINVAL;
  if (len < 0 || (len && (!y || !lambda || !y_inf || !out)))
    return fail(c, EMRKC_EINVAL, "exponential_euler_step: bad arguments");
  int rc = use(c);
  if (rc) return rc;
  if (!len) return EMRKC_OK;
  k_expeuler<<<grid_for(len), kThreads, 0, c->stream>>>(out, y, eta, lambda, y_inf, len);
  GK(c, cudaGetLastError());
  GK(c, cudaStreamSynchronize(c->stream));
  return EMRKC_OK;
}

int emrkc_rkc_iteration(emrkc_vctx* c, double t, const double* y, int64_t len, double dt,
                        emrkc_rhs_fn f, void* f_ctx, int32_t s, double epsilon, double* out,
                        int32_t* bad_stage) {
  if (!c) return EMRKC_EINVAL;
  if (!f || !y || !out || len < 1) return fail(c, EMRKC_EINVAL, "rkc_iteration: bad arguments");
  int rc = use(c);
  if (rc) return rc;
  CallbackRhs r;
  r.c = c;
  r.f = f;
  r.ctx = f_ctx;
  r.counter = nullptr;
  int32_t dummy = 0;
  rc = rkc_iter(c, t, y, len, dt, r, s, epsilon, out, bad_stage, &dummy);
  if (!rc) GK(c, cudaStreamSynchronize(c->stream));
  return rc;
}

int emrkc_averaged_force(emrkc_vctx* c, double t, const double* y, int64_t len, double eta,
                         const emrkc_split_rhs* rhs, int32_t m, int32_t variant, double epsilon,
                         double* out, int32_t* bad_stage) {
  if (!c) return EMRKC_EINVAL;
  if (!y || !out || len < 1) return fail(c, EMRKC_EINVAL, "averaged_force_emrkc: bad arguments");
  if (variant != EMRKC_VARIANT_STANDARD && variant != EMRKC_VARIANT_PROGRESSIVE)
    return fail(c, EMRKC_EINVAL, "averaged_force_emrkc: unknown variant %d", variant);
  int rc = use(c);
  if (rc) return rc;
  rc = averaged(c, t, y, len, eta, rhs, m, variant, epsilon, out, bad_stage);
  if (!rc) GK(c, cudaStreamSynchronize(c->stream));
  return rc;
}

int emrkc_averaged_force_mrkc(emrkc_vctx* c, double t, const double* y, int64_t len, double eta,
                              const emrkc_split_rhs* rhs, int32_t m, double epsilon, double* out,
                              int32_t* bad_stage) {
  if (!c) return EMRKC_EINVAL;
  if (!y || !out || len < 1) return fail(c, EMRKC_EINVAL, "averaged_force_mrkc: bad arguments");
  int rc = use(c);
  if (rc) return rc;
  rc = averaged(c, t, y, len, eta, rhs, m, 2, epsilon, out, bad_stage);
  if (!rc) GK(c, cudaStreamSynchronize(c->stream));
  return rc;
}

int emrkc_step_split(emrkc_vctx* c, double t, const double* y, int64_t len, double dt,
                     const emrkc_split_rhs* rhs, double epsilon, int32_t variant, double* out,
                     emrkc_step_report* report) {
  if (!c) return EMRKC_EINVAL;
  if (!y || !out || len < 1) return fail(c, EMRKC_EINVAL, "emrkc_step: bad arguments");
  if (variant != EMRKC_VARIANT_STANDARD && variant != EMRKC_VARIANT_PROGRESSIVE)
    return fail(c, EMRKC_EINVAL, "emrkc_step: unknown variant %d", variant);
  int rc = use(c);
  if (rc) return rc;
  rc = step_split(c, t, y, len, dt, rhs, epsilon, variant, out, report);
  if (!rc) GK(c, cudaStreamSynchronize(c->stream));
  return rc;
}

int emrkc_mrkc_step_split(emrkc_vctx* c, double t, const double* y, int64_t len, double dt,
                          const emrkc_split_rhs* rhs, double epsilon, double* out,
                          emrkc_step_report* report) {
  if (!c) return EMRKC_EINVAL;
  if (!y || !out || len < 1) return fail(c, EMRKC_EINVAL, "mrkc_step: bad arguments");
  int rc = use(c);
  if (rc) return rc;
  rc = step_split(c, t, y, len, dt, rhs, epsilon, 2, out, report);
  if (!rc) GK(c, cudaStreamSynchronize(c->stream));
  return rc;
}

int emrkc_estimate_spectral_radius(emrkc_vctx* c, double t, const double* y, int64_t len,
                                   emrkc_rhs_fn f, void* f_ctx, const double* v0, double rho0,
                                   emrkc_rho_result* out, double* v_out) {
  if (!c) return EMRKC_EINVAL;
  if (!f || !y || !out || len < 1)
    return fail(c, EMRKC_EINVAL, "estimate_spectral_radius: bad arguments");
  int rc = use(c);
  if (rc) return rc;
  constexpr double kEps = 1e-8, kTol = 1e-2;
  constexpr int kMaxIters = 50;
  Scratch sc(c);
  double* v = sc.get(len);
  double* fy = sc.get(len);
  double* fz = sc.get(len);
  double* z = sc.get(len);
  if (!v || !fy || !fz || !z) return fail(c, EMRKC_ENOMEM, "estimate_spectral_radius: out of memory");
  if (v0) {
    GK(c, cudaMemcpyAsync(v, v0, sizeof(double) * len, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    const std::vector<double> hv = seeded_direction(len);
    GK(c, cudaMemcpyAsync(v, hv.data(), sizeof(double) * len, cudaMemcpyHostToDevice, c->stream));
    GK(c, cudaStreamSynchronize(c->stream));
  }
  double nv = 0.0, ny = 0.0;
  if ((rc = norm2(c, v, len, &nv))) return rc;
  if (nv == 0.0) return fail(c, EMRKC_EINVAL, "estimate_spectral_radius: v0 must be nonzero");
  if ((rc = norm2(c, y, len, &ny))) return rc;
  const double delta = std::max(ny, kEps) * kEps;
  if (f(f_ctx, t, y, fy, len, c->stream)) return fail(c, EMRKC_ECALLBACK, "rhs callback failed");
  emrkc_rho_result r{};
  r.safety = 1.05;
  r.converged = 1;
  double rho = rho0, rho_old = 0.0;
  int it = 0;
  while (it == 0 || std::abs(rho - rho_old) >= kTol * rho) {
    if (it >= kMaxIters) {
      r.converged = 0;
      break;
    }
    rho_old = rho;
    const double q = delta / nv;
    k_zaxpy<<<grid_for(len), kThreads, 0, c->stream>>>(z, y, q, v, len);
    GK(c, cudaGetLastError());
    if (f(f_ctx, t, z, fz, len, c->stream)) return fail(c, EMRKC_ECALLBACK, "rhs callback failed");
    k_sub<<<grid_for(len), kThreads, 0, c->stream>>>(v, fz, fy, len);
    GK(c, cudaGetLastError());
    if ((rc = norm2(c, v, len, &nv))) return rc;
    if (nv < 1e-300) {  // locally null operator (P/src/spectral.cpp:61-66)
      r.rho = 0.0;
      r.iterations = it + 1;
      *out = r;
      if (v_out)
        GK(c, cudaMemcpyAsync(v_out, v, sizeof(double) * len, cudaMemcpyDeviceToDevice, c->stream));
      GK(c, cudaStreamSynchronize(c->stream));
      return EMRKC_OK;
    }
    rho = nv / delta;
    ++it;
  }
  r.rho = rho * r.safety;
  r.iterations = it;
  *out = r;
  if (v_out)
    GK(c, cudaMemcpyAsync(v_out, v, sizeof(double) * len, cudaMemcpyDeviceToDevice, c->stream));
  GK(c, cudaStreamSynchronize(c->stream));
  return EMRKC_OK;
}

}  // extern "C"
