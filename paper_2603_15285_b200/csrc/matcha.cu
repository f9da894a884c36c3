// matcha.cu -- host side of libmatcha: handle, FP64 table construction, C-ABI entry points and the
// align orchestration (App. C alternation around Algorithm 1, chunked over particles, one stream).
//
// Tables are computed here in double precision (own Gauss-Legendre Newton solve and normalised
// associated-Legendre recurrence; no code is shared with oracle/) and cast to the handle precision.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

using namespace matcha;

struct matcha_ctx {
  matcha_config_t cfg;
  int device = 0;
  int num_sms = 148;
  bool fp64 = false;
  bool use_tc = true;  // tcgen05 path for stage 2 (FP32 handles)
  size_t rsz = 4;  // sizeof(real)
  int R = 0, L = 0, Lq = 0, nth = 0, nph = 0, Jh = 0, ncf = 0;
  void* d_node = nullptr;
  void* d_tw = nullptr;
  void* d_pw = nullptr;     // m-major Legendre weights [Jh][pw_stride]
  int* d_pw_moff = nullptr;
  void* d_pwp = nullptr;    // parity-split Legendre weights [Jh][pwp_stride]
  int* d_pwp_off = nullptr; // [L+1][2] offsets of the (m, parity of l - m) blocks
  int pwp_stride = 0;
  void* d_dft = nullptr;    // parity-split cos/sin table of the folded ring DFT
  int Kh = 0, MP = 0, pw_stride = 0;
  int tcP = 0;              // plane slots of the tensor-core ring kernel (0 = SIMT ring kernel)
  int tcNR = 64;            // its rings per tile
  int* ws_tclist = nullptr; // its ring-list workspace when the list does not fit shared memory
  PairDesc* d_pairs = nullptr;
  void* d_pair_lnc = nullptr;
  RunDesc* d_runs = nullptr;
  void* d_run_lnc = nullptr;
  int* d_flags = nullptr;
  // align workspace (sized by max_batch)
  void* ws_F = nullptr;
  void* ws_M = nullptr;
  void* ws_H = nullptr;
  void* ws_G = nullptr;        // stage-1 ring coefficients of one sub-batch (L2-sized)
  int64_t gws_particles = 0;
  void* ws_euler = nullptr;
  void* ws_score = nullptr;
  int32_t* ws_idx = nullptr;
  int32_t* ws_best = nullptr;
  // host-buffer path
  float* ws_vols[2] = {nullptr, nullptr};
  void* ws_poses = nullptr;
  float* ws_ref = nullptr;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr};
  cudaEvent_t ev_used[2] = {nullptr, nullptr};
  int64_t launches = 0;
  std::string err;
  // stage 5 (translation): workspaces, allocated on first use
  void* ws_Fhat = nullptr;   // complex [mb][N][N][N/2+1]  f~: 2-D spectra of the particles' z-planes
  void* ws_FhatZ = nullptr;  // complex [mb][N][N][N/2+1]  F^ = z FFT of f~ (f3, FP32 fast path: once per chunk)
  bool fz_ready = false;     // ws_FhatZ holds the current chunk's F^
  void* ws_Xhat = nullptr;   // complex [mb][N][N][N/2+1]  rho~: 2-D spectra of the rotated references' planes
  void* ws_rho = nullptr;    // real [mb][N^3]             rotated references
  void* ws_peak = nullptr;   // real [mb]
  void* ws_win = nullptr;    // real [mb][window_scratch_reals(N, W)]: Y1 (z correlation) + the c window
  int ws_win_W = -1;
  void* ws_grid = nullptr;   // large coarse grids (f1): [chunk] x so3_large_workspace_bytes
  size_t ws_grid_bytes = 0;
  int* ws_tint = nullptr;    // int [mb][3]: integer window peaks (upsampled subpixel)
  void* ws_ups = nullptr;    // [mb] x ups_scratch_bytes(N, kappa): upsampled-DFT scratch
  int ws_ups_kappa = -1;
  bool trans_fast = false;   // FP32 and N in {32, 64, 96, 128}: compile-time FFTs, rotation fused into rho's transform
  float* ws_refpad = nullptr;  // zero-padded plane stacks of the references (texture sources of the fused rotation)
  int refpad_pitch = 0;        // floats per row
  cudaTextureObject_t tex_ref[kMaxTemplates] = {};
  cudaTextureObject_t* d_tex = nullptr;  // device copy of tex_ref
  // multi-template alignment
  void* ws_Hs = nullptr;     // complex [kMaxTemplates][ncoef][R] reference coefficients
  void* ws_cand = nullptr;   // real [kMaxTemplates][mb][8] per-template poses
  int* ws_tsel = nullptr;    // int [mb] selected template per particle
  void* ws_Rt = nullptr;     // matcha_reconstruct workspace: pose matrices + per-(class, half) particle lists
  int64_t ws_Rt_n = 0;       // bytes
  // ball-harmonic radial basis: tables for ball_lambda, workspaces
  double ball_lambda = -1;
  int ball_kmax = 0;
  std::vector<int> ball_K;   // |K_l|, l = 0..L
  void* d_ballB = nullptr;   // real [L+1][Kmax][R]
  int* d_ballK = nullptr;    // int [L+1]
  void* ws_Fb = nullptr;     // complex [mb][ncoef][R] (Kmax <= R) particle ball coefficients
  void* ws_Hb = nullptr;     // complex [ncoef][R] reference ball coefficients
  void* ws_euler1 = nullptr; // real [mb][3]
  // CUDA-graph replay of matcha_align_batch (matcha_set_graphs): the launch sequence of a call is captured once its
  // arguments repeat and replayed while they stay the same
  bool use_graphs = false;
  struct AlignKey {
    const float* vols;
    int64_t B;
    const float* ref;
    const void* ref_coeffs;
    matcha_params_t params;
    void* poses;
    cudaStream_t stream;
  };
  AlignKey last_key{};
  bool last_valid = false;
  cudaGraphExec_t graph_exec = nullptr;
  int64_t graph_launches = 0;
  // per-stage event tracing
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> ev_stage;  // stage of event pair k (events 2k, 2k+1)
  size_t ev_next = 0;
};

namespace {

matcha_status_t fail(matcha_handle_t h, matcha_status_t s, const std::string& msg) {
  if (h) h->err = msg;
  return s;
}

matcha_status_t cuda_fail(matcha_handle_t h, cudaError_t e, const char* where) {
  return fail(h, MATCHA_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define MATCHA_CUDA(h, expr)                          \
  do {                                                \
    cudaError_t _e = (expr);                          \
    if (_e != cudaSuccess) return cuda_fail(h, _e, #expr); \
  } while (0)

// ---------------------------------------------------------------- FP64 tables (host)
// Gauss-Legendre nodes on [-1,1], ascending, by Newton iteration on P_n from Tricomi's initial guess.
void gl_nodes(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int k = 1; k <= n; ++k) {
    const double th = kPi * (4.0 * k - 1.0) / (4.0 * n + 2.0);
    double z = (1.0 - (n - 1.0) / (8.0 * n * n * n)) * std::cos(th);
    double dp = 1.0;
    for (int it = 0; it < 60; ++it) {
      double pm = 1.0, p = z;  // P_0, P_1
      for (int j = 1; j < n; ++j) {
        const double pn = ((2.0 * j + 1.0) * z * p - j * pm) / (j + 1.0);
        pm = p;
        p = pn;
      }
      if (n == 1) { p = z; pm = 1.0; }
      dp = n * (pm - z * p) / (1.0 - z * z);
      const double dz = p / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-15 * std::max(1.0, std::fabs(z))) {
        // refresh derivative at the converged point
        double qm = 1.0, q = z;
        for (int j = 1; j < n; ++j) {
          const double qn = ((2.0 * j + 1.0) * z * q - j * qm) / (j + 1.0);
          qm = q;
          q = qn;
        }
        if (n == 1) { q = z; qm = 1.0; }
        dp = n * (qm - z * q) / (1.0 - z * z);
        break;
      }
    }
    x[n - k] = z;  // k = 1 is the largest root
    w[n - k] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

// normalised associated Legendre Pbar_lm(x) (Condon-Shortley phase), all 0 <= m <= l <= L
void plm_table(int L, double x, std::vector<double>& out) {
  out.assign(ncoef(L), 0.0);
  const double s = std::sqrt(std::max(0.0, (1.0 - x) * (1.0 + x)));
  double diag = 0.5 / std::sqrt(kPi);  // Pbar_00 = 1/sqrt(4 pi)
  for (int m = 0; m <= L; ++m) {
    if (m) diag *= -s * std::sqrt((2.0 * m + 1.0) / (2.0 * m));
    double p2 = diag;
    out[lm_index(m, m)] = p2;
    if (m == L) break;
    double p1 = x * std::sqrt(2.0 * m + 3.0) * diag;
    out[lm_index(m + 1, m)] = p1;
    for (int l = m + 2; l <= L; ++l) {
      const double l2 = (double)l * l, m2 = (double)m * m;
      const double a = std::sqrt((4.0 * l2 - 1.0) / (l2 - m2));
      const double b = std::sqrt(((l - 1.0) * (l - 1.0) - m2) / (4.0 * (l - 1.0) * (l - 1.0) - 1.0));
      const double p = a * (x * p1 - b * p2);
      out[lm_index(l, m)] = p;
      p2 = p1;
      p1 = p;
    }
  }
}

// spherical Bessel j_0..j_L at x by Miller's downward recurrence j_{n-1} = (2n+1)/x j_n - j_{n+1}, normalised by the
// identity sum_n (2n+1) j_n(x)^2 = 1 (robust near the zeros of j_0), the sign taken from the larger of
// j_0 = sin x / x and j_1 = sin x / x^2 - cos x / x; rescaled against overflow
void sph_bessel_all(int L, double x, std::vector<double>& j) {
  j.assign(L + 2, 0.0);
  if (x == 0.0) {
    j[0] = 1.0;
    return;
  }
  const int start = (int)std::max<double>(L + 2, x) + 60;
  std::vector<double> t(L + 2, 0.0);
  double jp = 0.0, jc = 1e-30, sum = (2.0 * start + 1.0) * jc * jc;
  for (int n = start; n >= 1; --n) {
    const double jm = (2.0 * n + 1.0) / x * jc - jp;
    jp = jc;
    jc = jm;
    sum += (2.0 * (n - 1) + 1.0) * jc * jc;
    if (n - 1 <= L + 1) t[n - 1] = jc;
    if (std::fabs(jc) > 1e150) {
      jc *= 1e-150;
      jp *= 1e-150;
      sum *= 1e-300;
      for (int q = n - 1; q <= L + 1; ++q) t[q] *= 1e-150;
    }
  }
  double sc = 1.0 / std::sqrt(sum);
  const double j0 = std::sin(x) / x, j1 = std::sin(x) / (x * x) - std::cos(x) / x;
  if (std::fabs(j0) >= std::fabs(j1) ? (j0 * t[0] < 0) : (j1 * t[1] < 0)) sc = -sc;
  for (int n = 0; n <= L + 1; ++n) j[n] = t[n] * sc;
}

double sph_bessel(int l, double x) {
  std::vector<double> j;
  sph_bessel_all(l, x, j);
  return j[l];
}

// positive roots of j_l below lam: sign changes on a 0.05 grid from x = l (the first root exceeds l), bisection
std::vector<double> sph_bessel_roots(int l, double lam) {
  std::vector<double> r;
  double x0 = std::max(0.5, (double)l), f0 = sph_bessel(l, x0);
  for (double x1 = x0 + 0.05; x0 <= lam; x1 += 0.05) {
    const double f1 = sph_bessel(l, x1);
    if (f0 == 0.0 || f0 * f1 < 0.0) {
      double a = x0, b = x1, fa = f0;
      for (int it = 0; it < 100 && b - a > 1e-15 * b; ++it) {
        const double m = 0.5 * (a + b), fm = sph_bessel(l, m);
        if ((fm < 0) == (fa < 0)) {
          a = m;
          fa = fm;
        } else {
          b = m;
        }
      }
      const double root = 0.5 * (a + b);
      if (root <= lam) r.push_back(root);
    }
    x0 = x1;
    f0 = f1;
  }
  return r;
}

template <typename T> void upload(void** dst, const std::vector<double>& src, cudaError_t& e) {
  std::vector<T> v(src.begin(), src.end());
  if (e == cudaSuccess) e = cudaMalloc(dst, sizeof(T) * std::max<size_t>(1, v.size()));
  if (e == cudaSuccess) e = cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
}

template <typename T> ShTables<T> sh_tables(matcha_handle_t h) {
  ShTables<T> t;
  t.node = (const cplx_t<T>*)h->d_node;
  t.tw = (const cplx_t<T>*)h->d_tw;
  t.pwm = (const T*)h->d_pw;
  t.pw_moff = h->d_pw_moff;
  t.pwp = (const T*)h->d_pwp;
  t.pwp_off = h->d_pwp_off;
  t.pwp_stride = h->pwp_stride;
  t.dft = (const cplx_t<T>*)h->d_dft;
  t.Kh = h->Kh;
  t.MP = h->MP;
  t.pw_stride = h->pw_stride;
  t.N = h->cfg.N;
  t.R = h->R;
  t.L = h->L;
  t.nth = h->nth;
  t.nph = h->nph;
  t.Jh = h->Jh;
  t.tcP = sizeof(T) == 4 ? h->tcP : 0;
  t.tcNR = h->tcNR;
  t.tc_list = h->ws_tclist;
  t.num_sms = h->num_sms;
  t.flags = h->d_flags;
  return t;
}

bool valid_params(const matcha_params_t* p, int LM, std::string& why) {
  if (!p) { why = "params is NULL"; return false; }
  if (p->n_bands < 1 || p->n_bands > 16) { why = "n_bands must be in [1,16]"; return false; }
  for (int j = 0; j < p->n_bands; ++j) {
    if (p->bands[j] < 1 || p->bands[j] > LM) { why = "band outside [1, L_M]"; return false; }
    if (j && p->bands[j] <= p->bands[j - 1]) { why = "bands must be strictly increasing"; return false; }
  }
  if (p->newton_iters < 0 || p->newton_iters > 64) { why = "newton_iters must be in [0,64]"; return false; }
  if (p->n_cand < 1 || p->n_cand > kMaxCand) { why = "n_cand must be in [1,32]"; return false; }
  if (p->oversample < 1 || p->oversample > 8) { why = "oversample must be in [1,8]"; return false; }
  if (p->n_alternations < 1 || p->n_alternations > 64) { why = "n_alternations must be in [1,64]"; return false; }
  if (p->upsample < 0) { why = "upsample must be >= 0"; return false; }
  if (p->radial != 0 && p->radial != 1) { why = "radial must be 0 (shells) or 1 (ball harmonics)"; return false; }
  return true;
}

template <typename T> NewtonArgs<T> newton_args(matcha_handle_t h) {
  NewtonArgs<T> a;
  std::memset(&a, 0, sizeof(a));
  a.runs = h->d_runs;
  a.run_lnc = (const T*)h->d_run_lnc;
  a.flags = h->d_flags;
  return a;
}

// RAII event pair around one stage launch (no-op unless profiling)
struct ProfScope {
  matcha_handle_t h;
  cudaStream_t s;
  size_t k = (size_t)-1;
  ProfScope(matcha_handle_t h_, int stage, cudaStream_t s_) : h(h_), s(s_) {
    if (!h->prof) return;
    k = h->ev_next++;
    while (h->ev_pool.size() < 2 * (k + 1)) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      h->ev_pool.push_back(e);
    }
    if (h->ev_stage.size() < k + 1) h->ev_stage.resize(k + 1);
    h->ev_stage[k] = stage;
    cudaEventRecord(h->ev_pool[2 * k], s);
  }
  ~ProfScope() {
    if (k != (size_t)-1) cudaEventRecord(h->ev_pool[2 * k + 1], s);
  }
};

}  // namespace

template <typename T>
static cudaError_t do_search(matcha_handle_t h, const void* M, int32_t L_M, int64_t B, int32_t L0, int32_t K,
                             int32_t nc, void* euler, void* score, int32_t* idx, cudaStream_t s) {
  SearchArgs<T> a;
  a.M = (const cplx_t<T>*)M;
  a.strideM = half_size(L_M);
  a.B = B;
  a.L0 = L0;
  a.K = K;
  a.ncand = nc;
  a.euler = (T*)euler;
  a.score = (T*)score;
  a.idx = idx;
  a.pairs = h->d_pairs;
  a.pair_lnc = (const T*)h->d_pair_lnc;
  a.flags = h->d_flags;
  return launch_so3_search<T>(a, s);
}

template <typename T>
static cudaError_t do_eval(matcha_handle_t h, const void* M, int32_t L_M, int64_t B, int32_t Q, int32_t L,
                           const void* euler, void* value, void* grad, void* hess, cudaStream_t s) {
  NewtonArgs<T> a = newton_args<T>(h);
  a.M = (const cplx_t<T>*)M;
  a.strideM = half_size(L_M);
  a.L_M = L_M;
  a.B = B;
  a.Q = Q;
  a.euler = (T*)euler;  // read only in eval mode
  a.value = (T*)value;
  a.grad = (T*)grad;
  a.hess = (T*)hess;
  a.L_eval = L;
  return launch_eval_corr<T>(a, grad != nullptr || hess != nullptr, s);
}

template <typename T>
static cudaError_t do_refine(matcha_handle_t h, const void* M, int32_t L_M, int64_t B, int32_t nc,
                             const matcha_params_t* p, void* euler, const int32_t* idx, void* score, int32_t* best,
                             cudaStream_t s) {
  NewtonArgs<T> a = newton_args<T>(h);
  a.M = (const cplx_t<T>*)M;
  a.strideM = half_size(L_M);
  a.L_M = L_M;
  a.B = B;
  a.Q = nc;
  a.euler = (T*)euler;
  a.idx = idx;
  a.nbands = p->n_bands;
  for (int j = 0; j < p->n_bands; ++j) a.bands[j] = p->bands[j];
  a.iters = p->newton_iters;
  a.tol_grad = p->tol_grad;
  a.tol_step = p->tol_step;
  a.tol_obj = p->tol_obj;
  a.score = (T*)score;
  a.best = best;
  return launch_newton_refine<T>(a, s);
}

// ---------------------------------------------------------------- stage 5 helpers
static matcha_status_t trans_prepare(matcha_handle_t h, int W, int kappa) {
  const int N = h->cfg.N;
  const int64_t nr = (int64_t)N * N * N, nc = (int64_t)N * N * (N / 2 + 1), mb = h->cfg.max_batch;
  if (!trans_supported(N, W, h->fp64))
    return fail(h, MATCHA_ERR_NOT_IMPLEMENTED, "translation: box/window exceed the stage-5 shared-memory limits");
  if (!h->ws_Fhat) {
    cudaError_t e = cudaMalloc(&h->ws_Fhat, 2 * h->rsz * nc * mb);
    if (e == cudaSuccess) e = cudaMalloc(&h->ws_Xhat, 2 * h->rsz * nc * mb);
    h->trans_fast = !h->fp64 && plane_fast_supported(N);
    if (e == cudaSuccess && !h->trans_fast) e = cudaMalloc(&h->ws_rho, h->rsz * nr * mb);
    if (e == cudaSuccess) e = cudaMalloc(&h->ws_peak, h->rsz * mb);
    if (e == cudaSuccess) e = cudaMalloc(&h->ws_euler1, 3 * h->rsz * mb);
    if (e != cudaSuccess) return fail(h, MATCHA_ERR_ALLOC, "translation workspace allocation failed");
    if (h->trans_fast) {
      int align = 32;
      cudaDeviceGetAttribute(&align, cudaDevAttrTexturePitchAlignment, h->device);
      const int af = std::max(1, align / (int)sizeof(float));
      h->refpad_pitch = (N + af - 1) / af * af;
      const size_t pad = (size_t)h->refpad_pitch * N * (N + 1);
      e = cudaMalloc((void**)&h->ws_refpad, sizeof(float) * pad * kMaxTemplates);
      if (e == cudaSuccess) e = cudaMalloc((void**)&h->d_tex, sizeof(cudaTextureObject_t) * kMaxTemplates);
      if (e != cudaSuccess) return fail(h, MATCHA_ERR_ALLOC, "translation reference texture allocation failed");
      for (int k = 0; k < kMaxTemplates; ++k) {
        cudaResourceDesc rd;
        std::memset(&rd, 0, sizeof(rd));
        rd.resType = cudaResourceTypePitch2D;
        rd.res.pitch2D.devPtr = h->ws_refpad + pad * k;
        rd.res.pitch2D.desc = cudaCreateChannelDesc<float>();
        rd.res.pitch2D.width = N;
        rd.res.pitch2D.height = (size_t)N * (N + 1);
        rd.res.pitch2D.pitchInBytes = sizeof(float) * (size_t)h->refpad_pitch;
        cudaTextureDesc td;
        std::memset(&td, 0, sizeof(td));
        td.addressMode[0] = td.addressMode[1] = cudaAddressModeBorder;  // border colour 0: zero outside the box
        td.filterMode = cudaFilterModePoint;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        e = cudaCreateTextureObject(&h->tex_ref[k], &rd, &td, nullptr);
        if (e != cudaSuccess) return cuda_fail(h, e, "translation: reference texture");
      }
      e = cudaMemcpy(h->d_tex, h->tex_ref, sizeof(cudaTextureObject_t) * kMaxTemplates, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return cuda_fail(h, e, "translation: texture table");
    }
  }
  if (kappa > 0 && h->trans_fast && !h->ws_FhatZ) {  // optional F^ cache of the upsampled path
    if (cudaMalloc(&h->ws_FhatZ, 2 * h->rsz * nc * mb) != cudaSuccess) {
      h->ws_FhatZ = nullptr;
      cudaGetLastError();
    }
    h->fz_ready = false;
  }
  if (h->ws_win_W < W) {
    if (h->ws_win) cudaFree(h->ws_win);
    h->ws_win = nullptr;
    h->ws_win_W = -1;
    if (cudaMalloc(&h->ws_win, h->rsz * window_scratch_reals(N, W) * mb) != cudaSuccess)
      return fail(h, MATCHA_ERR_ALLOC, "translation window scratch allocation failed");
    h->ws_win_W = W;
  }
  if (kappa > 0) {
    if (!ups_supported(N, kappa, h->fp64))
      return fail(h, MATCHA_ERR_NOT_IMPLEMENTED, "translation: upsample factor / box exceed the kernels' limits");
    if (!h->ws_tint && cudaMalloc((void**)&h->ws_tint, sizeof(int) * 3 * mb) != cudaSuccess)
      return fail(h, MATCHA_ERR_ALLOC, "translation: peak index allocation failed");
    if (h->ws_ups_kappa < kappa) {
      if (h->ws_ups) cudaFree(h->ws_ups);
      h->ws_ups = nullptr;
      h->ws_ups_kappa = -1;
      if (cudaMalloc(&h->ws_ups, ups_scratch_bytes(N, kappa, 2 * h->rsz) * mb) != cudaSuccess)
        return fail(h, MATCHA_ERR_ALLOC, "translation: upsampled-DFT scratch allocation failed");
      h->ws_ups_kappa = kappa;
    }
  }
  return MATCHA_OK;
}

// f~ (2-D plane spectra) of nb particle volumes into ws_Fhat (once per chunk: the particles do not change across
// alternations)
static matcha_status_t trans_fhat(matcha_handle_t h, const float* vols, int64_t nb, int W, int kappa,
                                  cudaStream_t s) {
  matcha_status_t st = trans_prepare(h, W, kappa);
  if (st != MATCHA_OK) return st;
  cudaError_t e = h->fp64 ? launch_plane_r2c<double, float>(vols, h->cfg.N, nb, (double2*)h->ws_Fhat, s)
                  : h->trans_fast
                      ? launch_plane_fft_f32(vols, nullptr, nullptr, nullptr, 0, h->cfg.N, nb, (float2*)h->ws_Fhat,
                                             false, s)
                      : launch_plane_r2c<float, float>(vols, h->cfg.N, nb, (float2*)h->ws_Fhat, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "translation: plane_r2c of the particles");
  h->launches++;
  h->fz_ready = false;  // a new chunk: its F^ is computed by the first upsampled update
  return MATCHA_OK;
}

// t = windowed argmax of c(t) = sum_x f(x) rho(x - t) for the rotations `euler` (stride estride)
// refs: float [nt][N^3]; tsel: the template of every particle (NULL when nt == 1)
static matcha_status_t trans_update(matcha_handle_t h, int64_t nb, const float* ref, int nt, const int* tsel,
                                    const void* euler, int estride, int W, int kappa, void* shifts, int sstride,
                                    void* peak, cudaStream_t s) {
  const int N = h->cfg.N;
  cudaError_t e;
  ProfScope ps(h, 5, s);
  matcha_status_t st = trans_prepare(h, W, kappa);
  if (st != MATCHA_OK) return st;
  if (h->trans_fast) {
    // rho~ straight from the reference texture: the rotated references never touch HBM
    const size_t pad = (size_t)h->refpad_pitch * N * (N + 1);
    for (int k = 0; k < nt; ++k) {
      e = launch_pad_ref(ref + (int64_t)k * N * N * N, N, h->refpad_pitch, h->ws_refpad + pad * k, s);
      if (e != cudaSuccess) return cuda_fail(h, e, "translation: pad_ref");
    }
    h->launches += nt - 1;
    e = launch_plane_fft_f32(nullptr, h->d_tex, tsel, (const float*)euler, estride, N, nb, (float2*)h->ws_Xhat, true,
                             s);
    if (e != cudaSuccess) return cuda_fail(h, e, "translation: plane_fft of rho");
  } else {
    e = h->fp64 ? launch_rotate_ref<double>(ref, N, (const double*)euler, estride, tsel, nb, (double*)h->ws_rho, s)
                : launch_rotate_ref<float>(ref, N, (const float*)euler, estride, tsel, nb, (float*)h->ws_rho, s);
    if (e != cudaSuccess) return cuda_fail(h, e, "translation: rotate_ref");
    e = h->fp64 ? launch_plane_r2c<double, double>((const double*)h->ws_rho, N, nb, (double2*)h->ws_Xhat, s)
                : launch_plane_r2c<float, float>((const float*)h->ws_rho, N, nb, (float2*)h->ws_Xhat, s);
    if (e != cudaSuccess) return cuda_fail(h, e, "translation: plane_r2c of rho");
  }
  int* tint = kappa > 0 ? h->ws_tint : nullptr;
  e = h->fp64 ? launch_window_zcorr<double>((const double2*)h->ws_Fhat, (const double2*)h->ws_Xhat, N, W, nb,
                                            (double*)h->ws_win, (double*)shifts, sstride, (double*)peak, tint, s)
              : launch_window_zcorr<float>((const float2*)h->ws_Fhat, (const float2*)h->ws_Xhat, N, W, nb,
                                           (float*)h->ws_win, (float*)shifts, sstride, (float*)peak, tint, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "translation: window_zcorr");
  h->launches += h->trans_fast ? 5 : 6;
  if (kappa > 0) {
    e = h->fp64 ? launch_upsampled<double>((const double2*)h->ws_Fhat, (double2*)h->ws_Xhat, N, kappa, nb, tint,
                                           h->ws_ups, (double*)shifts, sstride, (double*)peak, s)
                : launch_upsampled<float>((const float2*)h->ws_Fhat, (float2*)h->ws_Xhat, N, kappa, nb, tint,
                                          h->ws_ups, (float*)shifts, sstride, (float*)peak, s,
                                          (float2*)h->ws_FhatZ, h->fz_ready ? 2 : 1);
    if (e != cudaSuccess) return cuda_fail(h, e, "translation: upsampled DFT");
    h->fz_ready = h->ws_FhatZ != nullptr;
    h->launches += 4;
  }
  return MATCHA_OK;
}

// ball-harmonic tables for Lambda (reading C30: Lambda <= 0 -> pi (R - 1/2), the radial Nyquist of the R midpoint
// shells of the unit ball): B_l[k][i] = (1/R) rho_i^2 c_lk j_l(lambda_lk rho_i), c_lk = sqrt(2)/|j_{l+1}(lambda_lk)|
static matcha_status_t ball_prepare(matcha_handle_t h, double lam) {
  if (lam <= 0) lam = kPi * (h->R - 0.5);
  if (lam == h->ball_lambda) return MATCHA_OK;
  const int L = h->L, R = h->R;
  std::vector<std::vector<double>> roots(L + 1);
  int kmax = 0;
  for (int l = 0; l <= L; ++l) {
    roots[l] = sph_bessel_roots(l, lam);
    if ((int)roots[l].size() > R) roots[l].resize(R);
    kmax = std::max<int>(kmax, (int)roots[l].size());
  }
  if (kmax == 0) return fail(h, MATCHA_ERR_INVALID_ARG, "ball basis: Lambda below the first root of j_0");
  std::vector<double> tab((size_t)(L + 1) * kmax * R, 0.0), jv;
  std::vector<int> K(L + 1);
  for (int l = 0; l <= L; ++l) {
    K[l] = (int)roots[l].size();
    for (int k = 0; k < K[l]; ++k) {
      const double lk = roots[l][k];
      sph_bessel_all(l + 1, lk, jv);
      const double c = std::sqrt(2.0) / std::fabs(jv[l + 1]);
      for (int i = 0; i < R; ++i) {
        const double rho = (i + 0.5) / R;
        tab[((size_t)l * kmax + k) * R + i] = rho * rho / R * c * sph_bessel(l, lk * rho);
      }
    }
  }
  if (h->d_ballB) cudaFree(h->d_ballB);
  if (h->d_ballK) cudaFree(h->d_ballK);
  h->d_ballB = nullptr;
  h->d_ballK = nullptr;
  cudaError_t e = cudaSuccess;
  if (h->fp64) upload<double>(&h->d_ballB, tab, e);
  else upload<float>(&h->d_ballB, tab, e);
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->d_ballK, sizeof(int) * (L + 1));
  if (e == cudaSuccess) e = cudaMemcpy(h->d_ballK, K.data(), sizeof(int) * (L + 1), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(h, e, "ball basis tables");
  h->ball_K = K;
  h->ball_kmax = kmax;
  h->ball_lambda = lam;
  return MATCHA_OK;
}

static matcha_status_t ball_transform(matcha_handle_t h, const void* F, int64_t B, void* out, cudaStream_t s) {
  ProfScope ps(h, 7, s);
  cudaError_t e = h->fp64 ? launch_ball_transform<double>((const double2*)F, B, h->L, h->R, (const double*)h->d_ballB,
                                                          h->d_ballK, h->ball_kmax, (double2*)out, s)
                          : launch_ball_transform<float>((const float2*)F, B, h->L, h->R, (const float*)h->d_ballB,
                                                         h->d_ballK, h->ball_kmax, (float2*)out, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "ball_transform launch");
  h->launches += B > 0;
  return MATCHA_OK;
}

static matcha_status_t corr_ball(matcha_handle_t h, const void* Fb, const void* Hb, int64_t B, int L, void* M,
                                 cudaStream_t s) {
  ProfScope ps(h, 1, s);
  cudaError_t e = h->fp64 ? launch_corr_ball<double>((const double2*)Fb, (const double2*)Hb, B, L, h->L, h->d_ballK,
                                                     h->ball_kmax, (double2*)M, s)
                          : launch_corr_ball<float>((const float2*)Fb, (const float2*)Hb, B, L, h->L, h->d_ballK,
                                                    h->ball_kmax, (float2*)M, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "corr_ball launch");
  h->launches += B > 0;
  return MATCHA_OK;
}

// template norms live behind the per-particle template indices in ws_tsel (8-byte aligned: max_batch ints padded)
static double* tnorm(matcha_handle_t h) {
  return (double*)((char*)h->ws_tsel + ((sizeof(int) * h->cfg.max_batch + 7) / 8) * 8);
}

// App. C alternation around Algorithm 1 for particles [0, B) of `vols`, chunked by max_batch, against nt templates
// (refs float [nt][N^3]; ref_coeffs complex [nt][ncoef][R] or NULL): per alternation stage 1 once, stages 2-4 per
// template, the best-scoring template per particle (nt = 1: plain Algorithm 1), then the translation
// update against that template.  poses [B][pstride]: pstride 8, or 9 with the template index in column 8.
static matcha_status_t align_device(matcha_handle_t h, const float* vols, int64_t B, const float* refs, int nt,
                                    const void* ref_coeffs, const matcha_params_t* p, void* poses, int pstride,
                                    cudaStream_t s) {
  const int N = h->cfg.N;
  const int64_t n3 = (int64_t)N * N * N, hstride = (int64_t)h->ncf * h->R * 2 * h->rsz;
  const int LJ = p->bands[p->n_bands - 1], L0 = p->bands[0];
  const void* H = ref_coeffs;
  matcha_status_t st;
  if (!H) {
    if (nt > 1 && !h->ws_Hs && cudaMalloc(&h->ws_Hs, hstride * kMaxTemplates) != cudaSuccess)
      return fail(h, MATCHA_ERR_ALLOC, "align: template coefficient allocation failed");
    void* dst = nt == 1 ? h->ws_H : h->ws_Hs;
    st = matcha_sh_analysis(h, refs, nt, nullptr, dst, s);
    if (st != MATCHA_OK) return st;
    H = dst;
  }
  const bool ball = p->radial == 1;  // the correlation tensor from ball-harmonic coefficients
  if (ball) {
    if ((st = ball_prepare(h, p->ball_lambda)) != MATCHA_OK) return st;
    const size_t fbb = (size_t)h->cfg.max_batch * h->ncf * h->R * 2 * h->rsz;
    if (!h->ws_Fb && cudaMalloc(&h->ws_Fb, fbb) != cudaSuccess)
      return fail(h, MATCHA_ERR_ALLOC, "align: ball coefficient allocation failed");
    if (!h->ws_Hb && cudaMalloc(&h->ws_Hb, hstride * kMaxTemplates) != cudaSuccess)
      return fail(h, MATCHA_ERR_ALLOC, "align: reference ball coefficient allocation failed");
    // reference ball coefficients (Kmax <= R: the [nt][ncoef][Kmax] block fits the [nt][ncoef][R] workspace)
    if ((st = ball_transform(h, H, nt, h->ws_Hb, s)) != MATCHA_OK) return st;
  }
  const int64_t hbstride = (int64_t)h->ncf * h->ball_kmax * 2 * h->rsz;
  const bool direct = nt == 1 && pstride == 8;  // gather straight into the caller's poses (bitwise as before)
  if (!direct) {
    const size_t cb = (size_t)h->rsz * 8 * h->cfg.max_batch * kMaxTemplates;
    if (!h->ws_cand && cudaMalloc(&h->ws_cand, cb) != cudaSuccess)
      return fail(h, MATCHA_ERR_ALLOC, "align: template pose allocation failed");
    if (!h->ws_tsel && cudaMalloc((void**)&h->ws_tsel, (sizeof(int) * h->cfg.max_batch + 7) / 8 * 8 +
                                                           sizeof(double) * kMaxTemplates) != cudaSuccess)
      return fail(h, MATCHA_ERR_ALLOC, "align: template selection allocation failed");
    cudaError_t e = h->fp64 ? launch_template_norms<double>((const double2*)H, nt, h->L, LJ, h->R, tnorm(h), s)
                            : launch_template_norms<float>((const float2*)H, nt, h->L, LJ, h->R, tnorm(h), s);
    if (e != cudaSuccess) return cuda_fail(h, e, "align: template norms");
    h->launches++;
  }
  const bool translate = p->shift_window > 0;
  const int T = translate ? p->n_alternations : 1;  // without a translation update the T passes are identical
  for (int64_t c0 = 0; c0 < B; c0 += h->cfg.max_batch) {
    const int64_t nb = std::min<int64_t>(h->cfg.max_batch, B - c0);
    char* pc = (char*)poses + c0 * pstride * h->rsz;
    for (int tau = 0; tau < T; ++tau) {
      const void* sh = (tau > 0 && translate) ? (const void*)(pc + 3 * h->rsz) : nullptr;
      cudaError_t e;
      {
      ProfScope ps(h, 0, s);
      if (h->fp64)
        e = launch_sh_analysis<double>(vols + c0 * n3, nb, (const double*)sh, pstride, sh_tables<double>(h),
                                       (double2*)h->ws_F, (double2*)h->ws_G, h->gws_particles, s);
      else
        e = launch_sh_analysis<float>(vols + c0 * n3, nb, (const float*)sh, pstride, sh_tables<float>(h),
                                      (float2*)h->ws_F, (float2*)h->ws_G, h->gws_particles, s);
      }
      if (e != cudaSuccess) return cuda_fail(h, e, "align: sh_analysis");
      h->launches++;
      if (ball && (st = ball_transform(h, h->ws_F, nb, h->ws_Fb, s)) != MATCHA_OK) return st;
      for (int k = 0; k < nt; ++k) {
        const void* Hk = (const char*)H + k * hstride;
        if (ball) st = corr_ball(h, h->ws_Fb, (const char*)h->ws_Hb + k * hbstride, nb, LJ, h->ws_M, s);
        else st = matcha_corr_coeffs(h, h->ws_F, Hk, nb, LJ, h->ws_M, s);
        if (st != MATCHA_OK) return st;
        if ((st = matcha_so3_search(h, h->ws_M, LJ, nb, L0, p->oversample, p->n_cand, h->ws_euler, h->ws_score,
                                    h->ws_idx, s)) != MATCHA_OK)
          return st;
        if ((st = matcha_newton_refine(h, h->ws_M, LJ, nb, p->n_cand, p, h->ws_euler, h->ws_idx, h->ws_score,
                                       h->ws_best, s)) != MATCHA_OK)
          return st;
        void* dst = direct ? (void*)pc : (void*)((char*)h->ws_cand + (size_t)k * nb * 8 * h->rsz);
        {
        ProfScope ps(h, 4, s);
        e = h->fp64 ? launch_gather_poses<double>((const double*)h->ws_euler, (const double*)h->ws_score, h->ws_best,
                                                  nb, p->n_cand, !translate, (double*)dst, s)
                    : launch_gather_poses<float>((const float*)h->ws_euler, (const float*)h->ws_score, h->ws_best, nb,
                                                 p->n_cand, !translate, (float*)dst, s);
        }
        if (e != cudaSuccess) return cuda_fail(h, e, "align: gather_poses");
        h->launches++;
      }
      if (!direct) {
        ProfScope ps(h, 4, s);
        e = h->fp64 ? launch_select_template<double>((const double*)h->ws_cand, tnorm(h), nt, nb, translate,
                                                     (double*)pc, pstride, h->ws_tsel, s)
                    : launch_select_template<float>((const float*)h->ws_cand, tnorm(h), nt, nb, translate, (float*)pc,
                                                    pstride, h->ws_tsel, s);
        if (e != cudaSuccess) return cuda_fail(h, e, "align: select_template");
        h->launches++;
      }
      if (translate) {
        if (tau == 0) {
          ProfScope ps(h, 5, s);
          st = trans_fhat(h, vols + c0 * n3, nb, p->shift_window, p->upsample, s);
          if (st != MATCHA_OK) return st;
        }
        // t^tau from the rotation just estimated (poses[b][0..2]) -> poses[b][3..5]
        st = trans_update(h, nb, refs, nt, nt > 1 ? h->ws_tsel : nullptr, pc, pstride, p->shift_window, p->upsample,
                          pc + 3 * h->rsz, pstride, h->ws_peak, s);
        if (st != MATCHA_OK) return st;
      }
    }
  }
  return MATCHA_OK;
}

extern "C" {

MATCHA_API matcha_status_t matcha_create(const matcha_config_t* cfg, matcha_handle_t* out) {
  if (!cfg || !out) return MATCHA_ERR_INVALID_ARG;
  *out = nullptr;
  if (cfg->N < 8 || cfg->N > 512 || (cfg->N & 7)) return MATCHA_ERR_INVALID_ARG;
  if (cfg->L_max < 1 || cfg->L_max > kMaxL) return MATCHA_ERR_DEGREE;
  if (cfg->quad_oversample < 1 || cfg->quad_oversample > 8) return MATCHA_ERR_INVALID_ARG;
  if (cfg->max_batch < 1) return MATCHA_ERR_INVALID_ARG;
  if (cfg->precision != MATCHA_FP32 && cfg->precision != MATCHA_FP64) return MATCHA_ERR_INVALID_ARG;
  matcha_handle_t h = new matcha_ctx();
  h->cfg = *cfg;
  cudaGetDevice(&h->device);
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
  if (const char* v = getenv("MATCHA_CORR_SIMT")) h->use_tc = !(v[0] == '1');
  h->fp64 = cfg->precision == MATCHA_FP64;
  h->rsz = h->fp64 ? 8 : 4;
  h->R = cfg->N / 2;
  h->L = cfg->L_max;
  h->Lq = cfg->quad_oversample * cfg->L_max;
  h->nth = h->Lq + 1;
  h->nph = 2 * h->Lq + 2;
  h->Jh = (h->nth + 1) / 2;
  h->ncf = ncoef(h->L);

  // quadrature tables (readings C4): nodes ascending, phi_k = 2 pi k / n_phi
  std::vector<double> x, w;
  gl_nodes(h->nth, x, w);
  std::vector<double> node(2 * h->nth), tw(2 * h->nph);
  for (int j = 0; j < h->nth; ++j) {
    node[2 * j] = x[j];
    node[2 * j + 1] = std::sqrt(std::max(0.0, (1.0 - x[j]) * (1.0 + x[j])));
  }
  for (int k = 0; k < h->nph; ++k) {
    tw[2 * k] = std::cos(2.0 * kPi * k / h->nph);
    tw[2 * k + 1] = std::sin(2.0 * kPi * k / h->nph);
  }
  // Legendre weights W_j Pbar_lm(x_j), m-major with each m block padded to a multiple of 4 (float4 tiles)
  std::vector<int> moff(h->L + 2, 0);
  for (int mm = 0; mm <= h->L; ++mm) moff[mm + 1] = moff[mm] + (h->L - mm + 4) / 4 * 4;
  h->pw_stride = moff[h->L + 1];
  std::vector<double> pw((size_t)h->Jh * h->pw_stride, 0.0), P;
  for (int j = 0; j < h->Jh; ++j) {
    plm_table(h->L, x[j], P);
    for (int l = 0; l <= h->L; ++l)
      for (int mm = 0; mm <= l; ++mm) pw[(size_t)j * h->pw_stride + moff[mm] + (l - mm)] = w[j] * P[lm_index(l, mm)];
  }
  // the same weights with each m block split by the parity of l - m (l = m + p, m + p + 2, ...), each part padded
  // to a multiple of 4: a thread tile of 4 same-parity degrees reads a single node-pair combination (G+ or G-)
  std::vector<int> poff(2 * (h->L + 1), 0);
  int pst = 0;
  for (int mm = 0; mm <= h->L; ++mm)
    for (int par = 0; par < 2; ++par) {
      const int cnt = (mm + par <= h->L) ? (h->L - mm - par) / 2 + 1 : 0;
      poff[2 * mm + par] = pst;
      pst += (cnt + 3) / 4 * 4;
    }
  h->pwp_stride = std::max(pst, 4);
  std::vector<double> pwp((size_t)h->Jh * h->pwp_stride, 0.0);
  for (int j = 0; j < h->Jh; ++j)
    for (int mm = 0; mm <= h->L; ++mm)
      for (int l = mm; l <= h->L; ++l) {
        const int par = (l - mm) & 1;
        pwp[(size_t)j * h->pwp_stride + poff[2 * mm + par] + (l - mm - par) / 2] =
            pw[(size_t)j * h->pw_stride + moff[mm] + (l - mm)];
      }
  // folded ring-DFT table: [k = 0..Kh][m = 0..L] (cos, sin)(m phi_k)
  const int Mp = h->nph / 2;
  h->Kh = (Mp - 1) / 2;
  h->MP = h->L + 1;
  std::vector<double> dft((size_t)2 * (h->Kh + 1) * h->MP, 0.0);
  for (int k = 0; k <= h->Kh; ++k)
    for (int mm = 0; mm <= h->L; ++mm) {
      const double ang = 2.0 * kPi * (double)((long)mm * k % h->nph) / h->nph;
      dft[2 * ((size_t)k * h->MP + mm)] = std::cos(ang);
      dft[2 * ((size_t)k * h->MP + mm) + 1] = std::sin(ang);
    }
  // stage-3/4 pair table, grouped by shell l0 = max(m,|n|): long l-runs first
  std::vector<PairDesc> pairs;
  std::vector<double> plnc;
  for (int k = 0; k <= h->L; ++k) {
    auto add = [&](int m, int n) {
      pairs.push_back(PairDesc{(int16_t)m, (int16_t)n, (int32_t)(half_offset(k) + (int64_t)m * (2 * k + 1) + (n + k))});
      const int p = std::abs(m + n);
      plnc.push_back(0.5 * (std::lgamma(2.0 * k + 1.0) - std::lgamma(p + 1.0) - std::lgamma(2.0 * k - p + 1.0)));
    };
    if (k == 0) { add(0, 0); continue; }
    for (int n = -k; n <= k; ++n) add(k, n);
    for (int m = 0; m < k; ++m) { add(m, -k); add(m, k); }
  }
  // stage-4 runs (RunDesc): each shell's pairs folded by the d symmetries, singles (k,+-k), (0,-k) alone
  std::vector<RunDesc> runs;
  std::vector<double> rlnc;
  auto hoff = [](int l, int m, int n) { return (int32_t)(half_offset(l) + (int64_t)m * (2 * l + 1) + (n + l)); };
  for (int k = 0; k <= h->L; ++k) {
    auto addr = [&](int mA, int nA, int mB, int nB) {
      const int32_t oA = hoff(k, mA, nA);
      runs.push_back(RunDesc{(int16_t)mA, (int16_t)nA, (int16_t)mB, (int16_t)nB, oA, mB >= 0 ? hoff(k, mB, nB) : oA});
      const int p = std::abs(mA + nA);
      rlnc.push_back(0.5 * (std::lgamma(2.0 * k + 1.0) - std::lgamma(p + 1.0) - std::lgamma(2.0 * k - p + 1.0)));
    };
    if (k == 0) { addr(0, 0, -1, 0); continue; }
    for (int n = -k + 1; n < 0; ++n) addr(k, n, -n, -k);
    for (int n = 0; n < k; ++n) addr(k, n, n, k);
    addr(k, k, -1, 0);
    addr(k, -k, -1, 0);
    addr(0, -k, -1, 0);
  }
  cudaError_t e = cudaSuccess;
  if (h->fp64) {
    upload<double>(&h->d_node, node, e);
    upload<double>(&h->d_tw, tw, e);
    upload<double>(&h->d_pw, pw, e);
    upload<double>(&h->d_pwp, pwp, e);
    upload<double>(&h->d_dft, dft, e);
    upload<double>(&h->d_pair_lnc, plnc, e);
    upload<double>(&h->d_run_lnc, rlnc, e);
  } else {
    upload<float>(&h->d_node, node, e);
    upload<float>(&h->d_tw, tw, e);
    upload<float>(&h->d_pw, pw, e);
    upload<float>(&h->d_pwp, pwp, e);
    upload<float>(&h->d_dft, dft, e);
    upload<float>(&h->d_pair_lnc, plnc, e);
    upload<float>(&h->d_run_lnc, rlnc, e);
  }
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->d_pwp_off, sizeof(int) * poff.size());
  if (e == cudaSuccess) e = cudaMemcpy(h->d_pwp_off, poff.data(), sizeof(int) * poff.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->d_pw_moff, sizeof(int) * moff.size());
  if (e == cudaSuccess) e = cudaMemcpy(h->d_pw_moff, moff.data(), sizeof(int) * moff.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->d_pairs, sizeof(PairDesc) * pairs.size());
  if (e == cudaSuccess) e = cudaMemcpy(h->d_pairs, pairs.data(), sizeof(PairDesc) * pairs.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->d_runs, sizeof(RunDesc) * runs.size());
  if (e == cudaSuccess) e = cudaMemcpy(h->d_runs, runs.data(), sizeof(RunDesc) * runs.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->d_flags, sizeof(int) * 4);
  if (e == cudaSuccess) e = cudaMemset(h->d_flags, 0, sizeof(int) * 4);
  // align workspace
  const size_t cb = 2 * h->rsz, mb = cfg->max_batch;
  if (e == cudaSuccess) e = cudaMalloc(&h->ws_F, cb * mb * h->ncf * h->R);
  if (e == cudaSuccess) e = cudaMalloc(&h->ws_M, cb * mb * half_size(h->L));
  if (e == cudaSuccess) e = cudaMalloc(&h->ws_H, cb * h->ncf * h->R);
  if (!h->fp64 && !(getenv("MATCHA_SH_SIMT") && getenv("MATCHA_SH_SIMT")[0] == '1')) {
    std::vector<float> xn(h->nth);
    for (int j = 0; j < h->nth; ++j) xn[j] = (float)x[j];
    int gl = 0;
    h->tcP = sh_tc_plane_slots(sh_tables<float>(h), xn, &h->tcNR, &gl);
    if (h->tcP > 0 && gl && e == cudaSuccess) e = cudaMalloc((void**)&h->ws_tclist, sizeof(int) * (size_t)h->num_sms * h->R * h->nth);
  }
  {
    const size_t per = cb * (size_t)h->R * h->nth * (h->L + 1);
    // ring-coefficient sub-batch of ~640 MB (1,000+ c2 particles): one persistent ring launch and one Legendre launch
    // per chunk; G then round-trips through HBM (+1.1 MB per c2 particle), which costs less than the per-launch setup
    // (TMEM allocation, DFT-matrix fill, weight-table staging) and wave tails of L2-sized (96 MB) sub-batches:
    // measured 1.825 -> 1.696 ms per 1,000 c2 particles.  MATCHA_GWS_MB overrides the budget (A/B switch).
    size_t gws_mb = 640;
    if (const char* v = getenv("MATCHA_GWS_MB")) gws_mb = std::max(1, atoi(v));
    h->gws_particles = std::max<int64_t>(32, (int64_t)((gws_mb << 20) / per));
    // persistent tensor-core ring kernel: whole waves of one particle per SM (at least one wave: for large L the
    // ring coefficients of a wave exceed L2 and round-trip through HBM, cheaper than idle SMs)
    if (h->tcP > 0) h->gws_particles = std::max<int64_t>(h->num_sms, h->gws_particles / h->num_sms * h->num_sms);
    h->gws_particles = std::min<int64_t>(h->gws_particles, cfg->max_batch);
    if (e == cudaSuccess) e = cudaMalloc(&h->ws_G, per * h->gws_particles);
  }
  if (e == cudaSuccess) e = cudaMalloc(&h->ws_euler, h->rsz * mb * kMaxCand * 3);
  if (e == cudaSuccess) e = cudaMalloc(&h->ws_score, h->rsz * mb * kMaxCand);
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->ws_idx, sizeof(int32_t) * mb * kMaxCand);
  if (e == cudaSuccess) e = cudaMalloc((void**)&h->ws_best, sizeof(int32_t) * mb);
  if (e != cudaSuccess) {
    matcha_destroy(h);
    return e == cudaErrorMemoryAllocation ? MATCHA_ERR_ALLOC : MATCHA_ERR_CUDA;
  }
  *out = h;
  return MATCHA_OK;
}

MATCHA_API matcha_status_t matcha_destroy(matcha_handle_t h) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  void* ptrs[] = {h->d_node, h->d_tw, h->d_pw, h->d_pw_moff, h->d_pwp, h->d_pwp_off, h->d_dft, h->d_pairs, h->d_pair_lnc, h->d_runs, h->d_run_lnc, h->d_flags, h->ws_F, h->ws_M, h->ws_H, h->ws_G, h->ws_tclist,
                  h->ws_euler, h->ws_score, h->ws_idx, h->ws_best, h->ws_vols[0], h->ws_vols[1], h->ws_poses,
                  h->ws_ref};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  for (int k = 0; k < kMaxTemplates; ++k)
    if (h->tex_ref[k]) cudaDestroyTextureObject(h->tex_ref[k]);
  for (void* q : {h->ws_Fhat, h->ws_FhatZ, h->ws_Xhat, h->ws_rho, h->ws_peak, h->ws_euler1, h->ws_win, (void*)h->ws_refpad,
                  (void*)h->ws_tint, h->ws_ups, h->ws_grid, (void*)h->d_tex, h->ws_Hs, h->ws_cand,
                  (void*)h->ws_tsel, h->ws_Rt, h->d_ballB, (void*)h->d_ballK, h->ws_Fb, h->ws_Hb})
    if (q) cudaFree(q);
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
  for (int i = 0; i < 2; ++i) {
    if (h->ev_copied[i]) cudaEventDestroy(h->ev_copied[i]);
    if (h->ev_used[i]) cudaEventDestroy(h->ev_used[i]);
  }
  delete h;
  return MATCHA_OK;
}

MATCHA_API int64_t matcha_coeff_count(matcha_handle_t h) { return h ? (int64_t)h->ncf * h->R : -1; }
MATCHA_API int64_t matcha_corr_count(int32_t L) { return L < 0 ? 0 : half_size(L); }
MATCHA_API int64_t matcha_launch_count(matcha_handle_t h) { return h ? h->launches : -1; }
MATCHA_API const char* matcha_last_error_string(matcha_handle_t h) { return h ? h->err.c_str() : "null handle"; }

MATCHA_API matcha_status_t matcha_profile_begin(matcha_handle_t h) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  h->prof = true;
  h->ev_next = 0;
  return MATCHA_OK;
}

MATCHA_API matcha_status_t matcha_profile_end(matcha_handle_t h, double* stage_ms, int64_t* stage_launches) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  double ms[MATCHA_NUM_STAGES] = {0};
  int64_t cnt[MATCHA_NUM_STAGES] = {0};
  if (h->ev_next) MATCHA_CUDA(h, cudaEventSynchronize(h->ev_pool[2 * (h->ev_next - 1) + 1]));
  for (size_t k = 0; k < h->ev_next; ++k) {
    float t = 0.f;
    MATCHA_CUDA(h, cudaEventElapsedTime(&t, h->ev_pool[2 * k], h->ev_pool[2 * k + 1]));
    ms[h->ev_stage[k]] += t;
    cnt[h->ev_stage[k]] += 1;
  }
  h->prof = false;
  h->ev_next = 0;
  for (int i = 0; i < MATCHA_NUM_STAGES; ++i) {
    if (stage_ms) stage_ms[i] = ms[i];
    if (stage_launches) stage_launches[i] = cnt[i];
  }
  return MATCHA_OK;
}

MATCHA_API matcha_status_t matcha_get_status(matcha_handle_t h, void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  MATCHA_CUDA(h, cudaStreamSynchronize(s));
  int f = 0;
  MATCHA_CUDA(h, cudaMemcpy(&f, h->d_flags, sizeof(int), cudaMemcpyDeviceToHost));
  MATCHA_CUDA(h, cudaMemset(h->d_flags, 0, sizeof(int)));
  if (f & FLAG_NONFINITE) return fail(h, MATCHA_ERR_NONFINITE, "non-finite value produced on device");
  if (f & FLAG_OVERFLOW) return fail(h, MATCHA_ERR_OVERFLOW, "coarse-grid local-maximum list overflowed");
  if (f & FLAG_PLANES) return fail(h, MATCHA_ERR_OVERFLOW, "stage-1 plane window overflowed (shift too large)");
  return MATCHA_OK;
}

MATCHA_API matcha_status_t matcha_sh_analysis(matcha_handle_t h, const float* vols, int64_t B, const void* shifts,
                                              void* coeffs, void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || (B > 0 && (!vols || !coeffs))) return fail(h, MATCHA_ERR_INVALID_ARG, "sh_analysis: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  ProfScope ps(h, 0, s);
  if (h->fp64)
    e = launch_sh_analysis<double>(vols, B, (const double*)shifts, 3, sh_tables<double>(h), (double2*)coeffs,
                                   (double2*)h->ws_G, h->gws_particles, s);
  else
    e = launch_sh_analysis<float>(vols, B, (const float*)shifts, 3, sh_tables<float>(h), (float2*)coeffs,
                                  (float2*)h->ws_G, h->gws_particles, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "sh_analysis launch");
  h->launches += B > 0;
  return MATCHA_OK;
}

MATCHA_API matcha_status_t matcha_corr_coeffs(matcha_handle_t h, const void* f, const void* href, int64_t B,
                                              int32_t L, void* M, void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || (B > 0 && (!f || !href || !M))) return fail(h, MATCHA_ERR_INVALID_ARG, "corr_coeffs: bad arguments");
  if (L < 0 || L > h->L) return fail(h, MATCHA_ERR_DEGREE, "corr_coeffs: L > L_max");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  ProfScope ps(h, 1, s);
  if (h->fp64)
    e = launch_corr_coeffs<double>((const double2*)f, (const double2*)href, B, L, h->L, h->R, (double2*)M, s);
  else if (h->use_tc && corr_tc_supported(L, h->R))
    e = launch_corr_coeffs_tc((const float2*)f, (const float2*)href, B, L, h->L, h->R, (float2*)M, h->num_sms, s);
  else
    e = launch_corr_coeffs<float>((const float2*)f, (const float2*)href, B, L, h->L, h->R, (float2*)M, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "corr_coeffs launch");
  h->launches += B > 0;
  return MATCHA_OK;
}


MATCHA_API matcha_status_t matcha_so3_search(matcha_handle_t h, const void* M, int32_t L_M, int64_t B, int32_t L0,
                                             int32_t oversample, int32_t n_cand, void* euler, void* score,
                                             int32_t* grid_idx, void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || (B > 0 && (!M || !euler || !score || !grid_idx)))
    return fail(h, MATCHA_ERR_INVALID_ARG, "so3_search: bad arguments");
  if (L_M < 0 || L_M > h->L) return fail(h, MATCHA_ERR_DEGREE, "so3_search: L_M > L_max");
  if (L0 < 1 || L0 > L_M) return fail(h, MATCHA_ERR_CUTOFF, "so3_search: L0 outside [1, L_M]");
  if (oversample < 1 || oversample > 8 || n_cand < 1 || n_cand > kMaxCand)
    return fail(h, MATCHA_ERR_INVALID_ARG, "so3_search: oversample in [1,8], n_cand in [1,32]");
  if ((int64_t)oversample * (L0 + 1) * 4 * oversample * (L0 + 1) * oversample * (L0 + 1) >= (1ll << 31))
    return fail(h, MATCHA_ERR_INVALID_ARG, "so3_search: grid exceeds 2^31 nodes");
  cudaStream_t s = (cudaStream_t)stream;
  ProfScope ps(h, 2, s);
  if (so3_large_needed(L0, oversample, h->fp64)) {
    // three-pass search over a global grid workspace, in chunks of max_batch particles
    const int64_t mb = h->cfg.max_batch;
    const size_t per = so3_large_workspace_bytes(L0, oversample, n_cand, h->fp64);
    const size_t need = per * (size_t)std::min<int64_t>(mb, B);
    if (h->ws_grid_bytes < need) {
      if (h->ws_grid) cudaFree(h->ws_grid);
      h->ws_grid = nullptr;
      h->ws_grid_bytes = 0;
      if (cudaMalloc(&h->ws_grid, need) != cudaSuccess)
        return fail(h, MATCHA_ERR_ALLOC, "so3_search: coarse-grid workspace allocation failed");
      h->ws_grid_bytes = need;
    }
    for (int64_t c0 = 0; c0 < B; c0 += mb) {
      const int64_t nb = std::min<int64_t>(mb, B - c0);
      cudaError_t e;
      const size_t rs = h->rsz;
      if (h->fp64) {
        SearchArgs<double> a;
        a.M = (const double2*)((const char*)M + c0 * half_size(L_M) * 2 * rs);
        a.strideM = half_size(L_M); a.B = nb; a.L0 = L0; a.K = oversample; a.ncand = n_cand;
        a.euler = (double*)((char*)euler + c0 * n_cand * 3 * rs); a.score = (double*)((char*)score + c0 * n_cand * rs);
        a.idx = grid_idx + c0 * n_cand; a.pairs = h->d_pairs; a.pair_lnc = (const double*)h->d_pair_lnc;
        a.flags = h->d_flags;
        e = launch_so3_search_large<double>(a, h->ws_grid, s);
      } else {
        SearchArgs<float> a;
        a.M = (const float2*)((const char*)M + c0 * half_size(L_M) * 2 * rs);
        a.strideM = half_size(L_M); a.B = nb; a.L0 = L0; a.K = oversample; a.ncand = n_cand;
        a.euler = (float*)((char*)euler + c0 * n_cand * 3 * rs); a.score = (float*)((char*)score + c0 * n_cand * rs);
        a.idx = grid_idx + c0 * n_cand; a.pairs = h->d_pairs; a.pair_lnc = (const float*)h->d_pair_lnc;
        a.flags = h->d_flags;
        e = launch_so3_search_large<float>(a, h->ws_grid, s);
      }
      if (e != cudaSuccess) return cuda_fail(h, e, "so3_search (large grid) launch");
      h->launches += 3;
    }
    return MATCHA_OK;
  }
  cudaError_t e = h->fp64 ? do_search<double>(h, M, L_M, B, L0, oversample, n_cand, euler, score, grid_idx, s)
                          : do_search<float>(h, M, L_M, B, L0, oversample, n_cand, euler, score, grid_idx, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "so3_search launch");
  h->launches += B > 0;
  return MATCHA_OK;
}


MATCHA_API matcha_status_t matcha_eval_corr(matcha_handle_t h, const void* M, int32_t L_M, int64_t B, int32_t Q,
                                            int32_t L, const void* euler, void* value, void* grad, void* hess,
                                            void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || Q < 1 || Q > 1024 || (B > 0 && (!M || !euler || !value)))
    return fail(h, MATCHA_ERR_INVALID_ARG, "eval_corr: bad arguments");
  if (L_M < 0 || L_M > h->L) return fail(h, MATCHA_ERR_DEGREE, "eval_corr: L_M > L_max");
  if (L < 0 || L > L_M) return fail(h, MATCHA_ERR_CUTOFF, "eval_corr: L > L_M");
  cudaStream_t s = (cudaStream_t)stream;
  ProfScope ps(h, 3, s);
  cudaError_t e = h->fp64 ? do_eval<double>(h, M, L_M, B, Q, L, euler, value, grad, hess, s)
                          : do_eval<float>(h, M, L_M, B, Q, L, euler, value, grad, hess, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "eval_corr launch");
  h->launches += B > 0;
  return MATCHA_OK;
}


MATCHA_API matcha_status_t matcha_newton_refine(matcha_handle_t h, const void* M, int32_t L_M, int64_t B,
                                                int32_t n_cand, const matcha_params_t* params, void* euler,
                                                const int32_t* grid_idx, void* score, int32_t* best, void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || n_cand < 1 || n_cand > kMaxCand || (B > 0 && (!M || !euler || !score || !best)))
    return fail(h, MATCHA_ERR_INVALID_ARG, "newton_refine: bad arguments");
  if (L_M < 0 || L_M > h->L) return fail(h, MATCHA_ERR_DEGREE, "newton_refine: L_M > L_max");
  std::string why;
  if (!valid_params(params, L_M, why)) return fail(h, MATCHA_ERR_CUTOFF, "newton_refine: " + why);
  cudaStream_t s = (cudaStream_t)stream;
  ProfScope ps(h, 3, s);
  cudaError_t e = h->fp64 ? do_refine<double>(h, M, L_M, B, n_cand, params, euler, grid_idx, score, best, s)
                          : do_refine<float>(h, M, L_M, B, n_cand, params, euler, grid_idx, score, best, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "newton_refine launch");
  h->launches += B > 0;
  return MATCHA_OK;
}

MATCHA_API matcha_status_t matcha_translation_update(matcha_handle_t h, const float* vols, int64_t B,
                                                     const float* ref, const void* euler, int32_t window,
                                                     int32_t upsample, void* shifts, void* peak, void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || (B > 0 && (!vols || !ref || !euler || !shifts)))
    return fail(h, MATCHA_ERR_INVALID_ARG, "translation_update: bad arguments");
  if (window < 0 || window > h->cfg.N / 4) return fail(h, MATCHA_ERR_WINDOW, "translation_update: W > N/4");
  if (upsample < 0 || (upsample > 0 && !ups_supported(h->cfg.N, upsample, h->fp64)))
    return fail(h, MATCHA_ERR_INVALID_ARG, "translation_update: upsample factor outside the supported range");
  if (!trans_supported(h->cfg.N, window, h->fp64))
    return fail(h, MATCHA_ERR_NOT_IMPLEMENTED, "translation_update: box too large for the stage-5 kernels");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n3 = (int64_t)h->cfg.N * h->cfg.N * h->cfg.N;
  for (int64_t c0 = 0; c0 < B; c0 += h->cfg.max_batch) {
    const int64_t nb = std::min<int64_t>(h->cfg.max_batch, B - c0);
    matcha_status_t st = trans_fhat(h, vols + c0 * n3, nb, window, upsample, s);
    if (st != MATCHA_OK) return st;
    st = trans_update(h, nb, ref, 1, nullptr, (const char*)euler + c0 * 3 * h->rsz, 3, window, upsample,
                      (char*)shifts + c0 * 3 * h->rsz, 3, peak ? (char*)peak + c0 * h->rsz : h->ws_peak, s);
    if (st != MATCHA_OK) return st;
  }
  return MATCHA_OK;
}


MATCHA_API matcha_status_t matcha_set_graphs(matcha_handle_t h, int32_t enable) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  h->use_graphs = enable != 0;
  if (!h->use_graphs && h->graph_exec) {
    cudaGraphExecDestroy(h->graph_exec);
    h->graph_exec = nullptr;
  }
  h->last_valid = false;
  return MATCHA_OK;
}

static bool same_key(const matcha_ctx::AlignKey& a, const matcha_ctx::AlignKey& b) {
  return a.vols == b.vols && a.B == b.B && a.ref == b.ref && a.ref_coeffs == b.ref_coeffs && a.poses == b.poses &&
         a.stream == b.stream && std::memcmp(&a.params, &b.params, sizeof(matcha_params_t)) == 0;
}

MATCHA_API matcha_status_t matcha_align_batch(matcha_handle_t h, const float* vols, int64_t B, const float* ref,
                                              const void* ref_coeffs, const matcha_params_t* params, void* poses,
                                              void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || (B > 0 && (!vols || !poses))) return fail(h, MATCHA_ERR_INVALID_ARG, "align_batch: bad arguments");
  std::string why;
  if (!valid_params(params, h->L, why)) return fail(h, MATCHA_ERR_CUTOFF, "align_batch: " + why);
  if (!ref_coeffs && !ref) return fail(h, MATCHA_ERR_INVALID_ARG, "align_batch: need ref or ref_coeffs");
  if (params->shift_window > 0 && (!ref || params->shift_window > h->cfg.N / 4))
    return fail(h, MATCHA_ERR_WINDOW, "align_batch: shift window needs ref and W <= N/4");
  if (params->shift_window > 0 && !trans_supported(h->cfg.N, params->shift_window, h->fp64))
    return fail(h, MATCHA_ERR_NOT_IMPLEMENTED, "align_batch: box too large for the stage-5 kernels");
  if (params->shift_window > 0 && params->upsample > 0 && !ups_supported(h->cfg.N, params->upsample, h->fp64))
    return fail(h, MATCHA_ERR_NOT_IMPLEMENTED, "align_batch: upsample factor / box exceed the kernels' limits");
  cudaStream_t s = (cudaStream_t)stream;
  if (h->use_graphs && !h->prof && s) {
    matcha_ctx::AlignKey key{vols, B, ref, ref_coeffs, *params, poses, s};
    if (h->last_valid && same_key(key, h->last_key)) {
      if (!h->graph_exec) {
        // second identical call: capture the launch sequence (every workspace already exists) and instantiate it
        cudaGraph_t g = nullptr;
        const int64_t l0 = h->launches;
        MATCHA_CUDA(h, cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        matcha_status_t st = align_device(h, vols, B, ref, 1, ref_coeffs, params, poses, 8, s);
        cudaError_t e = cudaStreamEndCapture(s, &g);
        if (st != MATCHA_OK) {
          if (g) cudaGraphDestroy(g);
          return st;
        }
        if (e != cudaSuccess) return cuda_fail(h, e, "align_batch: graph capture");
        e = cudaGraphInstantiate(&h->graph_exec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return cuda_fail(h, e, "align_batch: graph instantiate");
        h->graph_launches = h->launches - l0;
        h->launches = l0;
      }
      MATCHA_CUDA(h, cudaGraphLaunch(h->graph_exec, s));
      h->launches += h->graph_launches;
      return MATCHA_OK;
    }
    if (h->graph_exec) {
      cudaGraphExecDestroy(h->graph_exec);
      h->graph_exec = nullptr;
    }
    h->last_key = key;
    h->last_valid = true;
  }
  return align_device(h, vols, B, ref, 1, ref_coeffs, params, poses, 8, s);
}

MATCHA_API matcha_status_t matcha_align_multi(matcha_handle_t h, const float* vols, int64_t B, const float* refs,
                                              int32_t n_templates, const void* ref_coeffs,
                                              const matcha_params_t* params, void* poses, void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || (B > 0 && (!vols || !poses))) return fail(h, MATCHA_ERR_INVALID_ARG, "align_multi: bad arguments");
  if (n_templates < 1 || n_templates > kMaxTemplates)
    return fail(h, MATCHA_ERR_INVALID_ARG, "align_multi: n_templates must be in [1, 16]");
  std::string why;
  if (!valid_params(params, h->L, why)) return fail(h, MATCHA_ERR_CUTOFF, "align_multi: " + why);
  if (!ref_coeffs && !refs) return fail(h, MATCHA_ERR_INVALID_ARG, "align_multi: need refs or ref_coeffs");
  if (params->shift_window > 0 && (!refs || params->shift_window > h->cfg.N / 4))
    return fail(h, MATCHA_ERR_WINDOW, "align_multi: shift window needs refs and W <= N/4");
  if (params->shift_window > 0 && !trans_supported(h->cfg.N, params->shift_window, h->fp64))
    return fail(h, MATCHA_ERR_NOT_IMPLEMENTED, "align_multi: box too large for the stage-5 kernels");
  if (params->shift_window > 0 && params->upsample > 0 && !ups_supported(h->cfg.N, params->upsample, h->fp64))
    return fail(h, MATCHA_ERR_NOT_IMPLEMENTED, "align_multi: upsample factor / box exceed the kernels' limits");
  return align_device(h, vols, B, refs, n_templates, ref_coeffs, params, poses, 9, (cudaStream_t)stream);
}

MATCHA_API matcha_status_t matcha_reconstruct(matcha_handle_t h, const float* vols, int64_t B, const void* poses,
                                              int32_t pose_stride, int32_t class_col, int32_t n_classes,
                                              int64_t first_index, void* sums, int32_t* counts, void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || (B > 0 && (!vols || !poses)) || !sums || !counts)
    return fail(h, MATCHA_ERR_INVALID_ARG, "reconstruct: bad arguments");
  if (pose_stride < 6 || n_classes < 1 || n_classes > 32 || class_col >= pose_stride || (class_col < 0 && n_classes != 1) ||
      (class_col >= 0 && class_col < 6) || first_index < 0)
    return fail(h, MATCHA_ERR_INVALID_ARG, "reconstruct: bad pose layout / class arguments");
  if (h->cfg.N % 8) return fail(h, MATCHA_ERR_INVALID_ARG, "reconstruct: N must be a multiple of 8");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t need = (int64_t)reconstruct_workspace_bytes(B, n_classes, h->rsz);
  if (h->ws_Rt_n < need) {
    if (h->ws_Rt) cudaFree(h->ws_Rt);
    h->ws_Rt = nullptr;
    h->ws_Rt_n = 0;
    if (cudaMalloc(&h->ws_Rt, need) != cudaSuccess)
      return fail(h, MATCHA_ERR_ALLOC, "reconstruct: workspace allocation failed");
    h->ws_Rt_n = need;
  }
  ProfScope ps(h, 6, s);
  cudaError_t e = h->fp64 ? launch_reconstruct<double>(vols, B, h->cfg.N, (const double*)poses, pose_stride, class_col,
                                                       n_classes, first_index, (double*)h->ws_Rt, (double*)sums,
                                                       counts, s)
                          : launch_reconstruct<float>(vols, B, h->cfg.N, (const float*)poses, pose_stride, class_col,
                                                      n_classes, first_index, (float*)h->ws_Rt, (float*)sums, counts,
                                                      s);
  if (e != cudaSuccess) return cuda_fail(h, e, "reconstruct launch");
  h->launches += B > 0 ? 3 : 2;
  return MATCHA_OK;
}

MATCHA_API int32_t matcha_ball_kmax(matcha_handle_t h, double lambda, int32_t* K_host) {
  if (!h) return -1;
  if (ball_prepare(h, lambda) != MATCHA_OK) return -1;
  if (K_host)
    for (int l = 0; l <= h->L; ++l) K_host[l] = h->ball_K[l];
  return h->ball_kmax;
}

MATCHA_API matcha_status_t matcha_ball_transform(matcha_handle_t h, const void* F, int64_t B, double lambda,
                                                 void* Fball, void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || (B > 0 && (!F || !Fball))) return fail(h, MATCHA_ERR_INVALID_ARG, "ball_transform: bad arguments");
  matcha_status_t st = ball_prepare(h, lambda);
  if (st != MATCHA_OK) return st;
  return ball_transform(h, F, B, Fball, (cudaStream_t)stream);
}

MATCHA_API matcha_status_t matcha_corr_coeffs_ball(matcha_handle_t h, const void* fball, const void* hball, int64_t B,
                                                   int32_t L, double lambda, void* M, void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || (B > 0 && (!fball || !hball || !M)))
    return fail(h, MATCHA_ERR_INVALID_ARG, "corr_coeffs_ball: bad arguments");
  if (L < 0 || L > h->L) return fail(h, MATCHA_ERR_DEGREE, "corr_coeffs_ball: L > L_max");
  matcha_status_t st = ball_prepare(h, lambda);
  if (st != MATCHA_OK) return st;
  return corr_ball(h, fball, hball, B, L, M, (cudaStream_t)stream);
}

MATCHA_API matcha_status_t matcha_synth_particles(matcha_handle_t h, uint64_t seed, int64_t first_index, int64_t B,
                                                  double snr, double shift_max, float* vols, double* truth,
                                                  void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || first_index < 0 || (B > 0 && !vols) || shift_max < 0)
    return fail(h, MATCHA_ERR_INVALID_ARG, "synth_particles: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  void* ws = nullptr;
  MATCHA_CUDA(h, cudaMallocAsync(&ws, synth_workspace_bytes(h->cfg.N, B), s));
  cudaError_t e = launch_synth_particles(seed, first_index, B, h->cfg.N, snr, shift_max, vols, truth, ws, s);
  cudaFreeAsync(ws, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "synth_particles launch");
  h->launches += 4 + (B > 0 ? 1 + (B + 65534) / 65535 : 0);
  return MATCHA_OK;
}

MATCHA_API matcha_status_t matcha_align_batch_host(matcha_handle_t h, const float* vols_host, int64_t B,
                                                   const float* ref_host, const matcha_params_t* params,
                                                   void* poses_host, void* stream) {
  if (!h) return MATCHA_ERR_INVALID_ARG;
  if (B < 0 || (B > 0 && (!vols_host || !poses_host)) || !ref_host)
    return fail(h, MATCHA_ERR_INVALID_ARG, "align_batch_host: bad arguments");
  std::string why;
  if (!valid_params(params, h->L, why)) return fail(h, MATCHA_ERR_CUTOFF, "align_batch_host: " + why);
  if (params->shift_window > h->cfg.N / 4) return fail(h, MATCHA_ERR_WINDOW, "align_batch_host: W > N/4");
  if (params->shift_window > 0 && !trans_supported(h->cfg.N, params->shift_window, h->fp64))
    return fail(h, MATCHA_ERR_NOT_IMPLEMENTED, "align_batch_host: box too large for the stage-5 kernels");
  if (params->shift_window > 0 && params->upsample > 0 && !ups_supported(h->cfg.N, params->upsample, h->fp64))
    return fail(h, MATCHA_ERR_NOT_IMPLEMENTED, "align_batch_host: upsample factor / box exceed the kernels' limits");
  cudaStream_t s = (cudaStream_t)stream;
  const int N = h->cfg.N;
  const int64_t n3 = (int64_t)N * N * N, mb = h->cfg.max_batch;
  // lazily allocate the double-buffered staging area and the copy stream
  if (!h->copy_stream) {
    MATCHA_CUDA(h, cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      MATCHA_CUDA(h, cudaMalloc((void**)&h->ws_vols[i], sizeof(float) * mb * n3));
      MATCHA_CUDA(h, cudaEventCreateWithFlags(&h->ev_copied[i], cudaEventDisableTiming));
      MATCHA_CUDA(h, cudaEventCreateWithFlags(&h->ev_used[i], cudaEventDisableTiming));
    }
    MATCHA_CUDA(h, cudaMalloc(&h->ws_poses, 8 * h->rsz * mb));
    MATCHA_CUDA(h, cudaMalloc((void**)&h->ws_ref, sizeof(float) * n3));
  }
  MATCHA_CUDA(h, cudaMemcpyAsync(h->ws_ref, ref_host, sizeof(float) * n3, cudaMemcpyHostToDevice, s));
  // reference coefficients once
  matcha_status_t st = matcha_sh_analysis(h, h->ws_ref, 1, nullptr, h->ws_H, s);
  if (st != MATCHA_OK) return st;
  const int64_t nchunks = (B + mb - 1) / mb;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int buf = (int)(c & 1);
    const int64_t c0 = c * mb, nb = std::min<int64_t>(mb, B - c0);
    // copy stream waits until compute has finished with this buffer, then uploads chunk c
    MATCHA_CUDA(h, cudaStreamWaitEvent(h->copy_stream, h->ev_used[buf], 0));
    MATCHA_CUDA(h, cudaMemcpyAsync(h->ws_vols[buf], vols_host + c0 * n3, sizeof(float) * nb * n3,
                                   cudaMemcpyHostToDevice, h->copy_stream));
    MATCHA_CUDA(h, cudaEventRecord(h->ev_copied[buf], h->copy_stream));
    MATCHA_CUDA(h, cudaStreamWaitEvent(s, h->ev_copied[buf], 0));
    st = align_device(h, h->ws_vols[buf], nb, h->ws_ref, 1, h->ws_H, params, h->ws_poses, 8, s);
    if (st != MATCHA_OK) return st;
    MATCHA_CUDA(h, cudaMemcpyAsync((char*)poses_host + c0 * 8 * h->rsz, h->ws_poses, 8 * h->rsz * nb,
                                   cudaMemcpyDeviceToHost, s));
    MATCHA_CUDA(h, cudaEventRecord(h->ev_used[buf], s));
  }
  MATCHA_CUDA(h, cudaStreamSynchronize(s));
  return MATCHA_OK;
}

}  // extern "C"
