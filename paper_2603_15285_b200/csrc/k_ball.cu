// k_ball.cu -- SURVEY f2: the paper's ball-harmonic radial basis with eigenvalue truncation (App. A.1,
// P:1215-1235) as a variant of stages 1 and 2.
//
// psi_klm(x) = c_lk j_l(lambda_lk |x|) Y_lm(x/|x|) on the unit ball (the box's inscribed ball, radius R = N/2 voxels),
// lambda_lk the k-th positive root of the spherical Bessel function j_l, c_lk = sqrt(2) / |j_{l+1}(lambda_lk)|
// (orthonormal), truncated to lambda_lk <= Lambda (the set K_l of P:1228-1233).  From the shell coefficients
// f_lm(r_i) of stage 1 (r_i = i - 1/2, rho_i = r_i / R), by the midpoint rule in rho (reading C30):
//   f^_klm = sum_i (1/R) rho_i^2 c_lk j_l(lambda_lk rho_i) f_lm(r_i)        (stage 1b, k_ball_transform)
//   sigma_lmn = A_l[m][n] = sum_{k in K_l} f^_klm conj(h^_kln)               (stage 2b, k_corr_ball)
// so rank(A_l) <= |K_l|: the correlation tensor is built directly from its rank-|K_l| factors.
// The radial tables B_l[k][i] = (1/R) rho_i^2 c_lk j_l(lambda_lk rho_i) are built on the host in FP64 (matcha.cu).
#include "common.cuh"

namespace matcha {

namespace {

constexpr int kThreads = 256;

constexpr int kPG = 16;  // particles per CTA: the per-degree table (or reference block) is staged once for all

// one CTA per (l, group of kPG particles): out[p][lm][k] = sum_i Bt[l][k][i] F[p][lm][i] for 0 <= m <= l, k < K_l
// (zero padding up to Kmax); the l table is staged once, F's l rows particle by particle
template <typename T>
__global__ void __launch_bounds__(kThreads) k_ball_transform(const cplx_t<T>* __restrict__ F, int64_t B, int Lmax,
                                                             int R, const T* __restrict__ Bt,
                                                             const int* __restrict__ Kl, int Kmax,
                                                             cplx_t<T>* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int l = blockIdx.x, K = Kl[l];
  const int ncf = ncoef(Lmax);
  cplx_t<T>* Fs = reinterpret_cast<cplx_t<T>*>(smem);  // [l+1][R]
  T* Bs = reinterpret_cast<T*>(Fs + (l + 1) * R);      // [R][Kmax] (transposed: lanes take consecutive k)
  const T* Bl = Bt + (int64_t)l * Kmax * R;
  for (int t = threadIdx.x; t < K * R; t += kThreads) {
    const int k = t / R, i = t - k * R;
    Bs[i * Kmax + k] = Bl[t];
  }
  for (int64_t p = (int64_t)blockIdx.y * kPG; p < min(B, (int64_t)(blockIdx.y + 1) * kPG); ++p) {
    const cplx_t<T>* Fp = F + (p * ncf + lm_index(l, 0)) * (int64_t)R;
    __syncthreads();  // the previous particle's rows are consumed
    for (int t = threadIdx.x; t < (l + 1) * R; t += kThreads) Fs[t] = Fp[t];
    __syncthreads();
    cplx_t<T>* o = out + (p * ncf + lm_index(l, 0)) * (int64_t)Kmax;
    for (int t = threadIdx.x; t < (l + 1) * Kmax; t += kThreads) {
      const int m = t / Kmax, k = t - m * Kmax;
      T ar = T(0), ai = T(0);
      if (k < K) {
        const cplx_t<T>* fr = Fs + m * R;
        const T* br = Bs + k;
        for (int i = 0; i < R; ++i) {
          const T b = br[i * Kmax];
          ar = fma(b, fr[i].x, ar);
          ai = fma(b, fr[i].y, ai);
        }
      }
      o[t] = mk<T>(ar, ai);
    }
  }
}

// one CTA per (l, group of kPG particles): M^l_mn = sum_{k < K_l} f^_klm conj(h^_kln), conj(h^_{k,l,n}) =
// (-1)^n h^_{k,l,|n|} for n < 0 (reality of h, reading C3; the radial transform is real); the conjugated reference
// block is staged once per CTA
template <typename T>
__global__ void __launch_bounds__(kThreads) k_corr_ball(const cplx_t<T>* __restrict__ Fb,
                                                        const cplx_t<T>* __restrict__ Hb, int64_t B, int L, int Lmax,
                                                        const int* __restrict__ Kl, int Kmax,
                                                        cplx_t<T>* __restrict__ M) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int l = L - (int)blockIdx.x, K = Kl[l], w = 2 * l + 1;
  const int ncf = ncoef(Lmax);
  cplx_t<T>* Fs = reinterpret_cast<cplx_t<T>*>(smem);  // [l+1][Kmax]
  cplx_t<T>* Hs = Fs + (l + 1) * Kmax;                  // [K][w]  conj(h^_kln)
  const cplx_t<T>* Hp = Hb + (int64_t)lm_index(l, 0) * Kmax;
  for (int t = threadIdx.x; t < K * w; t += kThreads) {
    const int n = t / K - l, k = t - (t / K) * K;
    const cplx_t<T> h = Hp[(int64_t)abs(n) * Kmax + k];
    Hs[k * w + n + l] = (n >= 0) ? mk<T>(h.x, -h.y) : ((n & 1) ? mk<T>(-h.x, -h.y) : h);
  }
  for (int64_t p = (int64_t)blockIdx.y * kPG; p < min(B, (int64_t)(blockIdx.y + 1) * kPG); ++p) {
    const cplx_t<T>* Fp = Fb + (p * ncf + lm_index(l, 0)) * (int64_t)Kmax;
    __syncthreads();
    for (int t = threadIdx.x; t < (l + 1) * Kmax; t += kThreads) Fs[t] = Fp[t];
    __syncthreads();
    cplx_t<T>* Mo = M + p * half_size(L) + half_offset(l);
    for (int o = threadIdx.x; o < (l + 1) * w; o += kThreads) {
      const int m = o / w, nn = o - m * w;
      T ar = T(0), ai = T(0);
      for (int k = 0; k < K; ++k) {
        const cplx_t<T> f = Fs[m * Kmax + k], h = Hs[k * w + nn];
        ar = fma(f.x, h.x, fma(-f.y, h.y, ar));
        ai = fma(f.x, h.y, fma(f.y, h.x, ai));
      }
      Mo[o] = mk<T>(ar, ai);
    }
  }
}

}  // namespace

template <typename T>
cudaError_t launch_ball_transform(const cplx_t<T>* F, int64_t B, int Lmax, int R, const T* Bt, const int* Kl, int Kmax,
                                  cplx_t<T>* out, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  const size_t bytes = sizeof(cplx_t<T>) * (size_t)(Lmax + 1) * R + sizeof(T) * (size_t)Kmax * R;
  if (bytes > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_ball_transform<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  const int64_t ng = (B + kPG - 1) / kPG;
  for (int64_t g0 = 0; g0 < ng; g0 += 65535) {
    const int64_t n = ng - g0 < 65535 ? ng - g0 : 65535;
    const int64_t b0 = g0 * kPG;
    k_ball_transform<T><<<dim3((unsigned)(Lmax + 1), (unsigned)n), kThreads, bytes, s>>>(
        F + b0 * (int64_t)ncoef(Lmax) * R, B - b0, Lmax, R, Bt, Kl, Kmax, out + b0 * (int64_t)ncoef(Lmax) * Kmax);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <typename T>
cudaError_t launch_corr_ball(const cplx_t<T>* Fb, const cplx_t<T>* Hb, int64_t B, int L, int Lmax, const int* Kl,
                             int Kmax, cplx_t<T>* M, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  const size_t bytes = sizeof(cplx_t<T>) * ((size_t)(L + 1) * Kmax + (size_t)Kmax * (2 * L + 1));
  if (bytes > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_corr_ball<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  const int64_t ng = (B + kPG - 1) / kPG;
  for (int64_t g0 = 0; g0 < ng; g0 += 65535) {
    const int64_t n = ng - g0 < 65535 ? ng - g0 : 65535;
    const int64_t b0 = g0 * kPG;
    k_corr_ball<T><<<dim3((unsigned)(L + 1), (unsigned)n), kThreads, bytes, s>>>(
        Fb + b0 * (int64_t)ncoef(Lmax) * Kmax, Hb, B - b0, L, Lmax, Kl, Kmax, M + b0 * half_size(L));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template cudaError_t launch_ball_transform<float>(const float2*, int64_t, int, int, const float*, const int*, int,
                                                  float2*, cudaStream_t);
template cudaError_t launch_ball_transform<double>(const double2*, int64_t, int, int, const double*, const int*, int,
                                                   double2*, cudaStream_t);
template cudaError_t launch_corr_ball<float>(const float2*, const float2*, int64_t, int, int, const int*, int, float2*,
                                             cudaStream_t);
template cudaError_t launch_corr_ball<double>(const double2*, const double2*, int64_t, int, int, const int*, int,
                                              double2*, cudaStream_t);

}  // namespace matcha
