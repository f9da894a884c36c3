// common.cuh -- shared device/host helpers of libmatcha (product path; no oracle code).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/matcha.h"

namespace matcha {

// ------------------------------------------------------------------ real / complex types
template <typename T> struct Cplx;
template <> struct Cplx<float> { using type = float2; };
template <> struct Cplx<double> { using type = double2; };
template <typename T> using cplx_t = typename Cplx<T>::type;

template <typename T> __host__ __device__ __forceinline__ cplx_t<T> mk(T x, T y) {
  cplx_t<T> r;
  r.x = x;
  r.y = y;
  return r;
}

// ------------------------------------------------------------------ index layouts
__host__ __device__ __forceinline__ int ncoef(int L) { return (L + 1) * (L + 2) / 2; }
__host__ __device__ __forceinline__ int lm_index(int l, int m) { return l * (l + 1) / 2 + m; }
// half-plane M: (l, m in [0,l], n in [-l,l]) at half_offset(l) + m(2l+1) + (n+l)
__host__ __device__ __forceinline__ int64_t half_offset(int l) { return (int64_t)l * (l + 1) * (4 * l - 1) / 6; }
__host__ __device__ __forceinline__ int64_t half_size(int L) { return half_offset(L + 1); }
// number of (m >= 0, n) pairs with max(m,|n|) <= L
__host__ __device__ __forceinline__ int pair_count(int L) { return (L + 1) * (2 * L + 1); }

constexpr double kPi = 3.14159265358979323846264338327950288;
constexpr int kMaxL = 128;
constexpr int kMaxCand = 32;
constexpr int kMaxTemplates = 16;  // multi-template alignment

// device error flags
enum : int { FLAG_NONFINITE = 1, FLAG_OVERFLOW = 2, FLAG_PLANES = 4 };

// Stage-4 pair descriptor: (m, n) with m >= 0, grouped by shell l0 = max(m,|n|) (long l-runs first).
// lnc = 1/2 ln C(2 l0, |m+n|) (seed normalisation), in double on the host.
struct PairDesc {
  int16_t m, n;
  int32_t off0;  // half-plane offset of M^{l0}_mn, l0 = max(m, |n|): half_offset(l0) + m (2 l0 + 1) + n + l0
};

// Stage-4 recurrence run: the l-run of pair A = (l0, nA) (mA = l0) and, when mB >= 0, of its symmetry partner B whose
// Wigner d equals A's up to a sign at every l and beta (d^l_{nm} = (-1)^{m-n} d^l_{mn}, d^l_{-n,-m} = d^l_{mn}):
//   nA in [0, l0):   B = (nA, l0),   d_B = (-1)^{l0-nA} d_A
//   nA in (-l0, 0):  B = (-nA, -l0), d_B = d_A
// (l0, +-l0) and (0, -l0) run alone (mB = -1).  Grouped by shell l0 ascending, so the runs of degree <= L are the
// first run_count(L).
struct RunDesc {
  int16_t mA, nA, mB, nB;
  int32_t offA, offB;  // half-plane offsets of M^{l0}_{mA nA}, M^{l0}_{mB nB} (offB = offA when alone)
};
__host__ __device__ __forceinline__ int run_count(int L) { return L * L + 3 * L + 1; }

// ------------------------------------------------------------------ kernel argument packs
template <typename T> struct ShTables {
  const cplx_t<T>* node;  // [n_theta] (cos th_j, sin th_j), x_j ascending
  const cplx_t<T>* tw;    // [n_phi] (cos phi_k, sin phi_k)
  const T* pwm;           // [Jh][pw_stride] W_j Pbar_lm(x_j), m-major rows: m block at pw_moff[m], l - m inside,
                          // each m block padded to a multiple of 4 (zeros); j < Jh = (n_theta+1)/2
  const int* pw_moff;     // [L+2] offsets of the m blocks (pw_moff[L+1] = pw_stride)
  const T* pwp;           // [Jh][pwp_stride] the same weights, (m, parity of l - m) blocks of l = m + par + 2 i
  const int* pwp_off;     // [L+1][2] offsets of those blocks (each padded to a multiple of 4)
  int pwp_stride;
  const cplx_t<T>* dft;   // [Kh+1][L+1]: (cos, sin)(m phi_k) for the folded ring DFT
  int N, R, L, nth, nph, Jh, Kh, MP, pw_stride;
  int tcP;                // plane slots of the tensor-core ring kernel (0 = SIMT ring kernel), FP32 only
  int tcNR;               // rings per tile of the tensor-core ring kernel (64, 32 or 16)
  int* tc_list;           // its per-CTA ring-list workspace [num_sms][R * nth] when the list leaves shared memory
  int num_sms;
  int* flags;
};

template <typename T> struct NewtonArgs {
  const cplx_t<T>* M;
  int64_t strideM;  // Mh(L_M)
  int L_M;
  int64_t B;
  int Q;                 // candidates (rotations) per particle
  T* euler;              // [B][Q][3] in/out
  const int32_t* idx;    // [B][Q] or null: <0 = inactive
  // eval mode outputs
  T* value;
  T* grad;
  T* hess;
  int L_eval;
  // refine mode
  int nbands;
  int bands[16];
  int iters;
  double tol_grad, tol_step, tol_obj;
  T* score;
  int32_t* best;
  const RunDesc* runs;
  const T* run_lnc;      // 1/2 ln C(2 l0, |mA+nA|) per run
  int* flags;
};

template <typename T> struct SearchArgs {
  const cplx_t<T>* M;
  int64_t strideM;
  int64_t B;
  int L0, K, ncand;
  T* euler;     // [B][ncand][3]
  T* score;     // [B][ncand]
  int32_t* idx; // [B][ncand]
  const PairDesc* pairs;
  const T* pair_lnc;
  int* flags;
};

// ------------------------------------------------------------------ launchers (explicitly instantiated)
template <typename T>
cudaError_t launch_sh_analysis(const float* vols, int64_t B, const T* shifts, int shift_stride, const ShTables<T>& tab,
                               cplx_t<T>* F, cplx_t<T>* Gws, int64_t gws_particles, cudaStream_t s);
template <typename T> size_t sh_ring_workspace_elems(const ShTables<T>& tab);  // complex elements per particle
template <typename T>
cudaError_t launch_corr_coeffs(const cplx_t<T>* F, const cplx_t<T>* H, int64_t B, int L, int Lmax, int R,
                               cplx_t<T>* M, cudaStream_t s);
template <typename T> cudaError_t launch_so3_search(const SearchArgs<T>& a, cudaStream_t s);
template <typename T> cudaError_t launch_eval_corr(const NewtonArgs<T>& a, bool derivs, cudaStream_t s);
template <typename T> cudaError_t launch_newton_refine(const NewtonArgs<T>& a, cudaStream_t s);
// per particle, the template whose pose scores highest relative to the template's norm (reading C29;
// ties -> lowest template index):
// cand [nt][B][8] poses per template -> poses [B][pstride] (columns 0..7 copied, column 8 = template index unless
// pstride < 9), tsel [B]; shifts (columns 3..5) are taken from `poses` itself when keep_shift
template <typename T>
cudaError_t launch_select_template(const T* cand, const double* tnorm, int nt, int64_t B, bool keep_shift, T* poses,
                                   int pstride, int* tsel, cudaStream_t s);
// ||H_{<=L}||_w of nt templates (reading C29), H complex [nt][ncoef(Lmax)][R] -> out double [nt]
template <typename T>
cudaError_t launch_template_norms(const cplx_t<T>* H, int nt, int Lmax, int L, int R, double* out, cudaStream_t s);
template <typename T>
cudaError_t launch_gather_poses(const T* euler, const T* score, const int32_t* best, int64_t B, int Q, bool zero_shift,
                                T* poses, cudaStream_t s);
size_t search_smem_bytes(int L0, int K, bool fp64);
// coarse grids too large for one CTA (L0 = 30 at K = 2): three passes over a global grid workspace of
// so3_large_workspace_bytes per particle
bool so3_large_needed(int L0, int K, bool fp64);
size_t so3_large_workspace_bytes(int L0, int K, int ncand, bool fp64);
template <typename T> cudaError_t launch_so3_search_large(const SearchArgs<T>& a, void* ws, cudaStream_t s);
int sh_tc_plane_slots(const ShTables<float>& tab, const std::vector<float>& xnode, int* nr, int* glist);
cudaError_t launch_sh_rings_tc(const float* vols, int64_t nb, const float* shifts, int shift_stride,
                               const ShTables<float>& tab, int P, float2* G, int* flags, int num_sms,
                               cudaStream_t st);
size_t corr_tc_smem_bytes(int L, int R);
bool corr_tc_supported(int L, int R);
cudaError_t launch_corr_coeffs_tc(const float2* F, const float2* H, int64_t B, int L, int Lmax, int R, float2* M,
                                  int num_sms, cudaStream_t s);
// tsel: per-particle template index into refs [T][N^3] (multi-template alignment) or NULL (one reference)
template <typename T>
cudaError_t launch_rotate_ref(const float* refs, int N, const T* euler, int estride, const int* tsel, int64_t nb, T* rho,
                              cudaStream_t s);
// stage 5 without an FFT library (k_trans.cu): mixed-radix factorisation of a transform length
struct FftRadix {
  int n, nst;
  int rad[16];
};
FftRadix fft_radix(int n);
bool trans_supported(int N, int W, bool fp64);  // shared-memory limits of the stage-5 kernels
template <typename T, typename Tin>
cudaError_t launch_plane_r2c(const Tin* vol, int N, int64_t nb, cplx_t<T>* out, cudaStream_t s);
// FP32 fast path (N = 32, 64, 96, 128): compile-time FFTs; rot = true fuses the rotation of the reference (read
// through `tex`, a 2-D texture over launch_pad_ref's zero-padded plane stack) into the transform of rho
bool plane_fast_supported(int N);
cudaError_t launch_plane_fft_f32(const float* vol, const cudaTextureObject_t* tex, const int* tsel,
                                 const float* euler, int estride, int N, int64_t nb, float2* out, bool rot,
                                 cudaStream_t s);
cudaError_t launch_pad_ref(const float* ref, int N, int pitch, float* pad, cudaStream_t s);
size_t window_scratch_reals(int N, int W);
template <typename T>
cudaError_t launch_window_zcorr(const cplx_t<T>* ft, const cplx_t<T>* rt, int N, int W, int64_t nb, T* scratch,
                                T* shifts, int sstride, T* peak, int* tint, cudaStream_t s);
// upsampled-DFT subpixel refinement around the integer peaks tint (overwrites rt with X = F^ conj(rho^))
int ups_points(int kappa);
bool ups_supported(int N, int kappa, bool fp64);
size_t ups_scratch_bytes(int N, int kappa, size_t csz);  // per particle
template <typename T>
cudaError_t launch_upsampled(const cplx_t<T>* ft, cplx_t<T>* rt, int N, int kappa, int64_t nb, const int* tint,
                             void* scratch, T* shifts, int sstride, T* peak, cudaStream_t s,
                             cplx_t<T>* fz = nullptr, int fz_mode = 0);
// fz: optional cache [nb][N][N][N/2+1] of F^ = the z FFT of f~ (FP32 compile-time-N path): fz_mode 1 computes and
// stores it with X, 2 reads it instead of transforming f~ again (the particles do not change across alternations)

// ball-harmonic radial transform and the correlation tensor from its rank-|K_l| factors (k_ball.cu);
// Bt real [Lmax+1][Kmax][R] radial table, Kl int [Lmax+1]; ball coefficients complex [B][ncoef(Lmax)][Kmax]
template <typename T>
cudaError_t launch_ball_transform(const cplx_t<T>* F, int64_t B, int Lmax, int R, const T* Bt, const int* Kl, int Kmax,
                                  cplx_t<T>* out, cudaStream_t s);
template <typename T>
cudaError_t launch_corr_ball(const cplx_t<T>* Fb, const cplx_t<T>* Hb, int64_t B, int L, int Lmax, const int* Kl,
                             int Kmax, cplx_t<T>* M, cudaStream_t s);

// matcha_synth_particles (k_synth.cu): the seeded synthetic workload on the device (bench/test infrastructure)
size_t synth_workspace_bytes(int N, int64_t B);
cudaError_t launch_synth_particles(uint64_t seed, int64_t first, int64_t B, int N, double snr, double shift_max,
                                   float* vols, double* truth, void* ws, cudaStream_t s);

// half-map sums of the aligned particles per class (k_recon.cu); Rt: workspace real [B][12]
template <typename T>
cudaError_t launch_reconstruct(const float* vols, int64_t B, int N, const T* poses, int pstride, int ccol, int ncls,
                               int64_t first, T* Rt, T* sums, int* counts, cudaStream_t s);
size_t reconstruct_workspace_bytes(int64_t B, int ncls, size_t rsz);  // Rt + per-(class, half) particle lists

}  // namespace matcha
