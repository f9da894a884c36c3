// k_corr.cu -- stage 2: the per-degree Wigner coefficient tensor.
//
// north_star stage (2); PAPER.md P:1311-1314 (sigma_{l m m'} = sum_k f_klm conj(h_klm')) and P:1319-1328
// (A_l = sum_k a_lk b_lk^*), in the shell form of reading C2:
//   M^l_mn = sum_i w_i f_lm(r_i) conj(h_ln(r_i)),  w_i = r_i^2,  0 <= m <= l, -l <= n <= l,
// with conj(h_{l,n}) = (-1)^n h_{l,|n|} for n < 0 (reality of h, reading C3).
// Per degree l this is the complex GEMM [(l+1) x R] . [R x (2l+1)], batched over particles.
//
// This is the SIMT version (FP64 handles, and degrees / shell counts the tensor-core kernel does not take): one CTA per
// (m block, l, particle) stages its rows of F^l [mb x R] and the weighted, conjugated, TRANSPOSED reference block
// Ht^l [R x (2l+1)] in shared memory (consecutive n on consecutive banks; F rows broadcast), in chunks of rc shells
// when a whole block does not fit (large R, FP64); each thread owns up to 4 outputs M^l_mn accumulated over the chunks.
#include <algorithm>

#include "common.cuh"

namespace matcha {

namespace {

constexpr int kThreads = 256;
constexpr int kOut = 4;  // outputs per thread

template <typename T>
__global__ void __launch_bounds__(kThreads) k_corr_coeffs(const cplx_t<T>* __restrict__ F,
                                                          const cplx_t<T>* __restrict__ H, int L, int Lmax, int R,
                                                          int mb, int rc, cplx_t<T>* __restrict__ M) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int l = L - (int)blockIdx.y;  // big blocks first
  const int m0 = blockIdx.x * mb;
  if (m0 > l) return;
  const int nm = min(mb, l + 1 - m0);
  const int64_t p = blockIdx.z;
  const int w = 2 * l + 1;
  const int ncf = ncoef(Lmax);
  cplx_t<T>* Fl = (cplx_t<T>*)smem;   // [nm][rc]
  cplx_t<T>* Ht = Fl + mb * rc;       // [rc][w]
  const cplx_t<T>* Fp = F + p * (int64_t)ncf * R + (int64_t)lm_index(l, m0) * R;
  const cplx_t<T>* Hl = H + (int64_t)lm_index(l, 0) * R;
  T ar[kOut], ai[kOut];
#pragma unroll
  for (int q = 0; q < kOut; ++q) ar[q] = ai[q] = T(0);
  for (int r0 = 0; r0 < R; r0 += rc) {
    const int nr = min(rc, R - r0);
    __syncthreads();
    for (int t = threadIdx.x; t < nm * nr; t += kThreads) {
      const int m = t / nr, i = t - m * nr;
      Fl[m * rc + i] = Fp[(int64_t)m * R + r0 + i];
    }
    for (int t = threadIdx.x; t < nr * w; t += kThreads) {
      const int n = t / nr - l, i = t % nr;  // read H coalesced along r
      const T r = (T)(r0 + i) + T(0.5), wr = r * r;
      const cplx_t<T> h = Hl[(size_t)abs(n) * R + r0 + i];
      cplx_t<T> v;
      if (n >= 0) v = mk<T>(wr * h.x, -wr * h.y);                  // w conj(h_{l,n})
      else v = (n & 1) ? mk<T>(-wr * h.x, -wr * h.y) : mk<T>(wr * h.x, wr * h.y);  // w (-1)^n h_{l,|n|}
      Ht[i * w + (n + l)] = v;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kOut; ++q) {
      const int o = threadIdx.x + q * kThreads;
      if (o < nm * w) {
        const int m = o / w, nn = o - m * w;
        const cplx_t<T>* fr = Fl + m * rc;
        T xr = ar[q], xi = ai[q];
#pragma unroll 4
        for (int i = 0; i < nr; ++i) {
          const cplx_t<T> f = fr[i], h = Ht[i * w + nn];
          xr = fma(f.x, h.x, xr);
          xr = fma(-f.y, h.y, xr);
          xi = fma(f.x, h.y, xi);
          xi = fma(f.y, h.x, xi);
        }
        ar[q] = xr;
        ai[q] = xi;
      }
    }
  }
  cplx_t<T>* Mo = M + p * half_size(L) + half_offset(l) + (int64_t)m0 * w;
#pragma unroll
  for (int q = 0; q < kOut; ++q) {
    const int o = threadIdx.x + q * kThreads;
    if (o < nm * w) Mo[o] = mk<T>(ar[q], ai[q]);
  }
}

// one CTA per (particle, l) when the whole block fits shared memory (all of c3 / c5): F^l and Ht^l staged once
template <typename T>
__global__ void __launch_bounds__(kThreads) k_corr_coeffs_whole(const cplx_t<T>* __restrict__ F,
                                                          const cplx_t<T>* __restrict__ H, int L, int Lmax, int R,
                                                          cplx_t<T>* __restrict__ M) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int l = L - (int)(blockIdx.x % (L + 1));  // big blocks first
  const int64_t p = blockIdx.x / (L + 1);
  const int w = 2 * l + 1;
  const int ncf = ncoef(Lmax);
  cplx_t<T>* Fl = (cplx_t<T>*)smem;   // [(l+1)][R]
  cplx_t<T>* Ht = Fl + (l + 1) * R;   // [R][w]
  const cplx_t<T>* Fp = F + p * (int64_t)ncf * R + (int64_t)lm_index(l, 0) * R;
  const cplx_t<T>* Hl = H + (int64_t)lm_index(l, 0) * R;
  for (int t = threadIdx.x; t < (l + 1) * R; t += kThreads) Fl[t] = Fp[t];
  for (int t = threadIdx.x; t < R * w; t += kThreads) {
    const int n = t / R - l, i = t % R;  // read H coalesced along r
    const T r = (T)i + T(0.5), wr = r * r;
    const cplx_t<T> h = Hl[(size_t)abs(n) * R + i];
    cplx_t<T> v;
    if (n >= 0) v = mk<T>(wr * h.x, -wr * h.y);                  // w conj(h_{l,n})
    else v = (n & 1) ? mk<T>(-wr * h.x, -wr * h.y) : mk<T>(wr * h.x, wr * h.y);  // w (-1)^n h_{l,|n|}
    Ht[i * w + (n + l)] = v;
  }
  __syncthreads();
  cplx_t<T>* Mo = M + p * half_size(L) + half_offset(l);
  for (int o = threadIdx.x; o < (l + 1) * w; o += kThreads) {
    const int m = o / w, nn = o - m * w;
    const cplx_t<T>* fr = Fl + m * R;
    T ar = T(0), ai = T(0);
#pragma unroll 4
    for (int i = 0; i < R; ++i) {
      const cplx_t<T> f = fr[i], h = Ht[i * w + nn];
      ar = fma(f.x, h.x, ar);
      ar = fma(-f.y, h.y, ar);
      ai = fma(f.x, h.y, ai);
      ai = fma(f.y, h.x, ai);
    }
    Mo[o] = mk<T>(ar, ai);
  }
}

}  // namespace

template <typename T>
cudaError_t launch_corr_coeffs(const cplx_t<T>* F, const cplx_t<T>* H, int64_t B, int L, int Lmax, int R,
                               cplx_t<T>* M, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  const size_t whole = sizeof(cplx_t<T>) * (size_t)R * ((L + 1) + (2 * L + 1));
  if (whole <= 200 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_corr_coeffs_whole<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)whole);
    if (e != cudaSuccess) return e;
    k_corr_coeffs_whole<T><<<(unsigned)(B * (L + 1)), kThreads, whole, s>>>(F, H, L, Lmax, R, M);
    return cudaGetLastError();
  }
  const int w = 2 * L + 1;
  const int mb = std::max(1, std::min(L + 1, kOut * kThreads / w));  // rows of the widest block per CTA
  const size_t cs = sizeof(cplx_t<T>), budget = 200 * 1024;
  int rc = R;
  while (rc > 1 && cs * (size_t)rc * (mb + w) > budget) rc = (rc + 1) / 2;
  const size_t bytes = cs * (size_t)rc * (mb + w);
  cudaError_t e = cudaFuncSetAttribute(k_corr_coeffs<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {  // gridDim.z <= 65535
    const int64_t nb = std::min<int64_t>(65535, B - b0);
    const dim3 grid((unsigned)((L + 1 + mb - 1) / mb), (unsigned)(L + 1), (unsigned)nb);
    k_corr_coeffs<T><<<grid, kThreads, bytes, s>>>(F + b0 * (int64_t)ncoef(Lmax) * R, H, L, Lmax, R, mb, rc,
                                                   M + b0 * half_size(L));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template cudaError_t launch_corr_coeffs<float>(const float2*, const float2*, int64_t, int, int, int, float2*,
                                               cudaStream_t);
template cudaError_t launch_corr_coeffs<double>(const double2*, const double2*, int64_t, int, int, int, double2*,
                                                cudaStream_t);

}  // namespace matcha
