/*
 * matcha.h -- C ABI of the B200-native Matcha hot path (arXiv 2603.15285, "Matcha, a
 * Multi-band Angular Template Matching Algorithm").  libmatcha.so, built for sm_100a.
 *
 * The method (Algorithm 1, plus the App. C alternation)
 * aligns each particle volume f to a reference h: argmax over g in SO(3) (and a shift t)
 * of the band-limited correlation C_L(g) = sum_{l<=L} sum_{m,n} conj(M^l_mn) D^l_mn(g)
 * (Eq. 4, with the conjugate placement of DESIGN.md reading C1).
 *
 * Conventions:
 *   - Volumes: float32 [N][N][N], x fastest (v[z][y][x]); centre c = (N-1)/2 per axis;
 *     trilinear interpolation of the zero-extended volume; N a multiple of 8, 8 <= N <= 512.
 *   - Euler angles (alpha, beta, gamma), ZYZ: g = r_z(alpha) r_y(beta) r_z(gamma) (Eq. 3,
 *     P:79-94), canonical ranges [0,2pi) x [0,pi] x [0,2pi); action (g o f)(x) = f(g^-1 x).
 *   - Shells r_i = i - 1/2, i = 1..R = N/2, weights w_i = r_i^2; angular quadrature: n_theta =
 *     L_q+1 Gauss-Legendre nodes, n_phi = 2 L_q + 2, L_q = quad_oversample * L_max.
 *   - Orthonormal complex SH with Condon-Shortley phase; f_{l,-m} = (-1)^m conj f_{lm}.
 *   - D^l_mn(a,b,g) = e^{-i m a} d^l_mn(b) e^{-i n g}, d^1_10 = -sin(b)/sqrt2.
 *   - "real" = float (MATCHA_FP32 handles) or double (MATCHA_FP64 handles); "complex" =
 *     interleaved (re, im) pairs of real.  Volumes are float32 in both precisions.
 *
 * Memory and ownership: every array argument is a DEVICE pointer (cudaMalloc / torch CUDA
 * tensor), contiguous, at least 16-byte aligned, owned by the caller, unless the argument
 * name ends in _host.  The library never frees caller memory; the handle owns only its
 * tables and workspace (allocated in matcha_create, sized by max_batch, freed in
 * matcha_destroy).  `stream` is a cudaStream_t (NULL = legacy default stream).
 *
 * Errors: argument checks run on the host before any launch and return a status
 * synchronously.  Launch failures return MATCHA_ERR_CUDA.  Device-side conditions
 * (non-finite values, candidate-list overflow) are recorded in a device flag and reported
 * by matcha_get_status().  No call synchronises the stream except matcha_get_status and
 * matcha_align_batch_host.  Results are bitwise reproducible for a given handle
 * configuration and input (fixed reduction orders, no floating-point atomics).
 * Thread safety: one host thread per handle at a time.
 */
#ifndef MATCHA_H_
#define MATCHA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define MATCHA_API __attribute__((visibility("default")))
#else
#define MATCHA_API
#endif

typedef struct matcha_ctx* matcha_handle_t;

typedef enum {
  MATCHA_OK = 0,
  MATCHA_ERR_INVALID_ARG = -1,   /* null pointer, B < 0, N odd or out of range, bad params */
  MATCHA_ERR_DEGREE = -2,        /* L > handle L_max, or L_max > 128 */
  MATCHA_ERR_CUTOFF = -3,        /* band > L_M, bands not strictly increasing, L0 > L_M */
  MATCHA_ERR_SHAPE = -4,         /* tensor shapes inconsistent with the handle */
  MATCHA_ERR_WINDOW = -5,        /* shift window W > N/4 */
  MATCHA_ERR_NONFINITE = -6,     /* a non-finite value was produced (device flag) */
  MATCHA_ERR_CUDA = -7,          /* CUDA runtime / launch error */
  MATCHA_ERR_ALLOC = -8,         /* device allocation failed */
  MATCHA_ERR_NOT_IMPLEMENTED = -9,
  MATCHA_ERR_OVERFLOW = -10      /* more coarse-grid local maxima than the candidate buffer holds */
} matcha_status_t;

typedef enum { MATCHA_FP32 = 0, MATCHA_FP64 = 1 } matcha_precision_t;

/* Handle configuration (host struct). */
typedef struct {
  int32_t N;               /* box edge (voxels), multiple of 8, 8..512 */
  int32_t L_max;           /* analysis degree L (= last band L_J), 1..128 */
  int32_t quad_oversample; /* q: L_q = q * L_max (reading C4; default 2) */
  int32_t max_batch;       /* particles per internal chunk of matcha_align_batch */
  int32_t precision;       /* matcha_precision_t */
} matcha_config_t;

/* Algorithm 1 / App. C parameters (host struct). */
typedef struct {
  int32_t n_bands;         /* J+1 */
  int32_t bands[16];       /* L_0 < L_1 < ... < L_J <= L_M; Newton runs at every band incl. L_0 */
  int32_t newton_iters;    /* M_iter Newton steps per band (default 1) */
  int32_t n_cand;          /* N_C candidates kept from the coarse search, 1..32 */
  int32_t oversample;      /* K, SO(3)-grid oversampling (default 2) */
  int32_t n_alternations;  /* T rotation/translation alternations (App. C); used only when
                              shift_window > 0 (without a translation update one rotation pass is run) */
  int32_t shift_window;    /* W: translation search window [-W,W]^3 voxels, W <= N/4; 0 = rotation only */
  int32_t upsample;        /* subpixel step of the translation update: 0 = per-axis parabola (reading C18);
                              kappa >= 1 = upsampled DFT (Guizar-Sicairos, App. C remark iii; reading C27):
                              the correlation's trigonometric interpolant on a 1/kappa grid over +-1.5 voxel around
                              the integer peak (kappa <= 21; 16 in SURVEY f3) */
  int32_t radial;          /* radial representation of stage 2: 0 = shells (reading C2, default);
                              1 = the paper's ball harmonics (App. A.1) with the eigenvalue cutoff
                              ball_lambda: M^l = sum_{k in K_l} f^_kl conj(h^_kl), rank <= |K_l| */
  double tol_grad;         /* early stop: ||grad|| < tol_grad*|C|; 0 = off */
  double tol_step;         /* early stop: ||delta|| < tol_step (rad); 0 = off */
  double tol_obj;          /* early stop: |dC| < tol_obj*|C|; 0 = off */
  double ball_lambda;      /* Lambda of the ball-harmonic truncation lambda_lk <= Lambda (unit-ball frequency);
                              <= 0: pi (R - 1/2), the radial Nyquist of the R midpoint shells (reading C30) */
} matcha_params_t;

/* Create a handle on the CURRENT CUDA device: builds the quadrature, Legendre and Wigner
   index tables in FP64 on the host, uploads them, allocates the align workspace. */
MATCHA_API matcha_status_t matcha_create(const matcha_config_t* cfg, matcha_handle_t* out);
MATCHA_API matcha_status_t matcha_destroy(matcha_handle_t h);

/* Sizes (elements of "complex"): ncoef(L_max) * R per particle; Mh(L) = (L+1)(L+2)(4L+3)/6. */
MATCHA_API int64_t matcha_coeff_count(matcha_handle_t h);
MATCHA_API int64_t matcha_corr_count(int32_t L);

/* Stage 1 -- shell spherical-harmonic analysis (north_star stage 1):
     f_lm(r_i) = sum_j W_j Pbar_lm(cos th_j) (2pi/n_phi) sum_k u(c + t + r_i w_jk) e^{-i m phi_k}
   vols: float32 [B][N][N][N]; shifts: real [B][3] (x,y,z voxels; shell centre c + t) or NULL (t = 0);
   coeffs (out): complex [B][ncoef(L_max)][R], index (l(l+1)/2 + m)*R + (i-1), 0 <= m <= l, unweighted. */
MATCHA_API matcha_status_t matcha_sh_analysis(matcha_handle_t h, const float* vols, int64_t B, const void* shifts,
                                              void* coeffs, void* stream);

/* Stage 2 -- Wigner coefficient tensor (north_star stage 2):
     M^l_mn = sum_i w_i f_lm(r_i) conj(h_ln(r_i)),   0 <= m <= l <= L, -l <= n <= l
   f: complex [B][ncoef(L_max)][R]; href: complex [ncoef(L_max)][R] (unweighted reference coefficients H,
   w_i applied inside); M (out): complex [B][Mh(L)] half plane, entry l(l+1)(4l-1)/6 + m(2l+1) + (n+l).
   Requires L <= L_max. */
MATCHA_API matcha_status_t matcha_corr_coeffs(matcha_handle_t h, const void* f, const void* href, int64_t B,
                                              int32_t L, void* M, void* stream);

/* Stage 3 -- coarse SO(3) search (north_star stage 3; Alg. 1 lines 1-2):
   C_{L0} on the grid n_beta = K(L0+1), n_alpha = n_gamma = 2K(L0+1), beta_j = (j+1/2)pi/n_beta,
   alpha_a = 2pi a/n_alpha, gamma_c = 2pi c/n_gamma (reading C9), evaluated per beta slice by a Wigner-d
   contraction and a 2-D DFT over (alpha, gamma); then the n_cand strongest strict local maxima (26
   neighbours; alpha, gamma periodic, beta clamped; ties -> lower linear index (j n_a + a) n_g + c) ranked by
   (score desc, index asc) (readings C10, C11).
   M: complex [B][Mh(L_M)], L0 <= L_M; euler (out): real [B][n_cand][3]; score (out): real [B][n_cand];
   grid_idx (out): int32 [B][n_cand], -1 (score -inf, euler 0) where fewer maxima exist. */
MATCHA_API matcha_status_t matcha_so3_search(matcha_handle_t h, const void* M, int32_t L_M, int64_t B, int32_t L0,
                                             int32_t oversample, int32_t n_cand, void* euler, void* score,
                                             int32_t* grid_idx, void* stream);

/* Evaluation of C_L, its gradient and Hessian in the Euler chart (Eq. 4) at Q
   rotations per particle -- the kernel behind stage 4, exported for parity tests.
   M: complex [B][Mh(L_M)], L <= L_M; euler: real [B][Q][3]; value (out): real [B][Q];
   grad (out): real [B][Q][3] (d/da, d/db, d/dg); hess (out): real [B][Q][6] (aa, bb, gg, ab, ag, bg).
   grad/hess may be NULL (value only). */
MATCHA_API matcha_status_t matcha_eval_corr(matcha_handle_t h, const void* M, int32_t L_M, int64_t B, int32_t Q,
                                            int32_t L, const void* euler, void* value, void* grad, void* hess,
                                            void* stream);

/* Stage 4 -- frequency-marching Newton refinement (north_star stage 4; Alg. 1 lines 3-8):
   for each band L_j in params->bands, params->newton_iters steps theta <- canon(theta - H_reg^-1 grad)
   with H_reg = H if -H > 0 else H - (lambda_max + 1e-6 ||H||_F) I (reading C13); then the final
   C_{L_J} of every candidate and the argmax (lowest index on ties).
   euler: real [B][n_cand][3] in/out; grid_idx: int32 [B][n_cand] or NULL (entries < 0 are inactive
   padding: not refined, score -inf); score (out): real [B][n_cand]; best (out): int32 [B]. */
MATCHA_API matcha_status_t matcha_newton_refine(matcha_handle_t h, const void* M, int32_t L_M, int64_t B,
                                                int32_t n_cand, const matcha_params_t* params, void* euler,
                                                const int32_t* grid_idx, void* score, int32_t* best, void* stream);

/* Stage 5 -- translation update (App. C; readings C17, C18): rho = g o h (trilinear rotation
   of the reference, zero outside), c(t) = sum_x f(x) rho((x - t) mod N) (the FFT correlation of P:1797, evaluated
   on the window from 2-D plane spectra: hand-written FFTs, no library), argmax over the window [-W,W]^3 (ties ->
   lowest window index, z-major); subpixel step: upsample = 0 -> parabola per axis clamped to 1/2; upsample = kappa
   -> upsampled DFT around the integer peak (see matcha_params_t.upsample; reading C27).
   vols: float32 [B][N^3]; ref: float32 [N^3]; euler: real [B][3]; shifts (out): real [B][3] (x,y,z
   voxels, particle frame: f ~ S_t(g o h)); peak (out): real [B] (c at the integer argmax, or c~ at the upsampled
   argmax), may be NULL.  Errors: WINDOW if W > N/4; NOT_IMPLEMENTED if the box/window/kappa exceed the kernels'
   shared-memory limits (FP32 boxes up to ~200 voxels). */
MATCHA_API matcha_status_t matcha_translation_update(matcha_handle_t h, const float* vols, int64_t B,
                                                     const float* ref, const void* euler, int32_t window,
                                                     int32_t upsample, void* shifts, void* peak, void* stream);

/* Whole path -- App. C alternation around Algorithm 1, chunked by max_batch:
   t = 0; repeat T times { stage 1 at centre c + t; stage 2; stage 3 (L_0); stage 4; if W > 0 stage 5 }.
   ref_coeffs: complex [ncoef(L_max)][R] reference coefficients H (e.g. broadcast from rank 0), or NULL to
   analyse `ref` here.  ref: float32 [N^3] (needed when ref_coeffs is NULL or W > 0).
   poses (out): real [B][8] = {alpha, beta, gamma, t_x, t_y, t_z, score, best_cand}. */
MATCHA_API matcha_status_t matcha_align_batch(matcha_handle_t h, const float* vols, int64_t B, const float* ref,
                                              const void* ref_coeffs, const matcha_params_t* params, void* poses,
                                              void* stream);

/* Ball-harmonic radial basis (App. A.1; reading C30).  psi_klm = c_lk j_l(lambda_lk rho)
   Y_lm on the box's inscribed ball (rho = r / R), lambda_lk the k-th positive root of j_l, c_lk = sqrt(2) /
   |j_{l+1}(lambda_lk)|, kept while lambda_lk <= lambda (lambda <= 0: pi (R - 1/2)).
   matcha_ball_kmax: fills K_host[0..L_max] with |K_l| (host array, may be NULL) and returns Kmax = max_l |K_l|
   (negative on error).
   matcha_ball_transform: shell coefficients F complex [B][ncoef(L_max)][R] (stage 1) -> ball coefficients
   Fball complex [B][ncoef(L_max)][Kmax], f^_klm = sum_i (1/R) rho_i^2 c_lk j_l(lambda_lk rho_i) f_lm(r_i) (midpoint
   rule, rho_i = (i - 1/2)/R), zero for k >= |K_l|.
   matcha_corr_coeffs_ball: M complex [B][Mh(L)] half plane, M^l_mn = sum_{k < |K_l|} f^_klm conj(h^_kln)
   (sigma_{l m m'} of P:1311-1314 with K_l; hball complex [ncoef(L_max)][Kmax]). */
MATCHA_API int32_t matcha_ball_kmax(matcha_handle_t h, double lambda, int32_t* K_host);
MATCHA_API matcha_status_t matcha_ball_transform(matcha_handle_t h, const void* F, int64_t B, double lambda,
                                                 void* Fball, void* stream);
MATCHA_API matcha_status_t matcha_corr_coeffs_ball(matcha_handle_t h, const void* fball, const void* hball, int64_t B,
                                                   int32_t L, double lambda, void* M, void* stream);

/* Multi-template alignment ("evaluate alignment against multiple candidate templates per
   iteration"): per alternation, stage 1 once per particle, stages 2-4 against every template, the template whose
   final C_{L_J} is highest (ties -> lowest template index) is kept, and the translation update (W > 0) rotates that
   template.  refs: float32 [n_templates][N^3] (needed when ref_coeffs is NULL or W > 0); ref_coeffs: complex
   [n_templates][ncoef(L_max)][R] or NULL; n_templates in [1, 16].
   poses (out): real [B][9] = {alpha, beta, gamma, t_x, t_y, t_z, score, best_cand, template}. */
MATCHA_API matcha_status_t matcha_align_multi(matcha_handle_t h, const float* vols, int64_t B, const float* refs,
                                              int32_t n_templates, const void* ref_coeffs,
                                              const matcha_params_t* params, void* poses, void* stream);

/* Reference update of subtomogram averaging (P:1184 half-set split; reading C28): the aligned
   particles summed in the reference frame per class and half set,
     sums[k][s][y] = sum_{p: class(p) = k, (first_index + p) mod 2 = s} f_p(g_p (y - c) + c + t_p)   (trilinear)
   vols: float32 [B][N^3]; poses: real [B][pose_stride] with {alpha, beta, gamma, t_x, t_y, t_z} in columns 0..5 and
   the class in column class_col (class_col < 0: one class; n_classes must then be 1; particles whose class is outside
   [0, n_classes) are skipped); first_index: global index of particle 0 (half set = parity of the global index).
   sums (out): real [n_classes][2][N^3]; counts (out): int32 [n_classes][2] (device).  The half maps are sums / counts;
   across GPUs all-reduce sums and counts first (paper_2603_15285_b200.dist.reconstruct_step).  Deterministic (fixed
   particle order per voxel, no atomics). */
MATCHA_API matcha_status_t matcha_reconstruct(matcha_handle_t h, const float* vols, int64_t B, const void* poses,
                                              int32_t pose_stride, int32_t class_col, int32_t n_classes,
                                              int64_t first_index, void* sums, int32_t* counts, void* stream);

/* Bench/test infrastructure: particles first_index .. first_index + B - 1 of the seeded
   synthetic workload generated on the device -- the Philox4x32-10 counter layout and Gaussian-blob phantom of
   gen/gen.c (reference blobs keyed 0x5EED): f_p = S_{t_p}(g_p o h) + eta_p, g_p Haar,
   t_p ~ U[-shift_max, shift_max]^3 (0: no shift), eta ~ N(0, P_ref / snr) (snr <= 0 or inf: noise-free).
   vols (out): float32 [B][N^3]; truth (out, may be NULL): double [B][12] = (g_p row-major, t_p).  Volumes agree with
   gen/gen.c to the last float ulp (device vs host exp/log).  Allocates a temporary workspace (stream-ordered). */
MATCHA_API matcha_status_t matcha_synth_particles(matcha_handle_t h, uint64_t seed, int64_t first_index, int64_t B,
                                                  double snr, double shift_max, float* vols, double* truth,
                                                  void* stream);

/* CUDA-graph replay of matcha_align_batch (off by default): when enabled, a call whose arguments (pointers, sizes,
   params, stream) repeat the previous call's is captured into a CUDA graph once and then replayed as a single
   launch while they stay the same (no per-kernel launch overhead for short shards).  Results are
   bitwise identical to the eager path.  Requires a non-default stream; disabled while profiling. */
MATCHA_API matcha_status_t matcha_set_graphs(matcha_handle_t h, int32_t enable);

/* End-to-end variant on HOST buffers: vols_host float32 [B][N^3] (pinned memory recommended), ref_host float32
   [N^3]; poses_host (out) real [B][8].  Copies chunks host->device on a second stream overlapped with compute,
   and synchronises before returning. */
MATCHA_API matcha_status_t matcha_align_batch_host(matcha_handle_t h, const float* vols_host, int64_t B,
                                                   const float* ref_host, const matcha_params_t* params,
                                                   void* poses_host, void* stream);

/* Synchronises `stream`, then reports (and clears) device-side error flags. */
MATCHA_API matcha_status_t matcha_get_status(matcha_handle_t h, void* stream);
MATCHA_API const char* matcha_last_error_string(matcha_handle_t h);
/* Number of kernel launches issued through this handle since creation (bench bookkeeping). */
MATCHA_API int64_t matcha_launch_count(matcha_handle_t h);

/* Per-stage tracing with CUDA events recorded on the launching stream around every stage launch.
   Stage ids: 0 sh_analysis, 1 corr_coeffs, 2 so3_search, 3 newton_refine/eval_corr, 4 pose gather / template
   selection, 5 translation_update, 6 reconstruct, 7 ball_transform.  matcha_profile_end synchronises on the last event and returns, per stage,
   the summed device milliseconds and the number of launches since matcha_profile_begin
   (stage_ms, stage_launches: host arrays of MATCHA_NUM_STAGES entries; either may be NULL). */
#define MATCHA_NUM_STAGES 8
MATCHA_API matcha_status_t matcha_profile_begin(matcha_handle_t h);
MATCHA_API matcha_status_t matcha_profile_end(matcha_handle_t h, double* stage_ms, int64_t* stage_launches);

#ifdef __cplusplus
}
#endif
#endif /* MATCHA_H_ */
