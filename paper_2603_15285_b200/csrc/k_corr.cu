// k_corr.cu -- stage 2: the per-degree Wigner coefficient tensor.
//
// north_star stage (2); PAPER.md P:1311-1314 (sigma_{l m m'} = sum_k f_klm conj(h_klm')) and P:1319-1328
// (A_l = sum_k a_lk b_lk^*), in the shell form of reading C2:
//   M^l_mn = sum_i w_i f_lm(r_i) conj(h_ln(r_i)),  w_i = r_i^2,  0 <= m <= l, -l <= n <= l,
// with conj(h_{l,n}) = (-1)^n h_{l,|n|} for n < 0 (reality of h, reading C3).
// Per degree l this is the complex GEMM [(l+1) x R] . [R x (2l+1)], batched over particles.
//
// This is the SIMT version (FP64 handles, and degrees / shell counts the tensor-core kernel does not take).  Per degree l
// the product is one real-shaped GEMM over all particles, rows (p, m), columns n, K = R shells, with the (weighted,
// conjugated) reference block Ht^l [R x (2l+1)] shared by every row.  One CTA computes a 64 x 64 complex tile of it:
// 16-shell chunks of the F rows and of Ht^l (built from H on the way in) are double-buffered in shared memory, k-major,
// and each thread accumulates a 4 x 4 register tile (6 shared loads per 64 FMAs).  Tiles of all degrees form one grid,
// large l first.
#include <algorithm>

#include "common.cuh"

namespace matcha {

namespace {

constexpr int kBM = 64, kBN = 64, kBK = 16;  // tile rows (p, m), tile columns n, shells per chunk
constexpr int kThreads = 256;                 // 16 x 16 threads, 4 x 4 outputs each

struct CorrTiles {
  int L;
  int64_t start[kMaxL + 2];  // start[i]: first tile of degree L - i; start[L + 1] = number of tiles
};

__host__ __device__ inline int col_tiles(int l) { return (2 * l + 1 + kBN - 1) / kBN; }

template <typename T>
__global__ void __launch_bounds__(kThreads) k_corr_tiled(const cplx_t<T>* __restrict__ F, const cplx_t<T>* __restrict__ H,
                                                         int64_t B, int Lmax, int R, const __grid_constant__ CorrTiles tl,
                                                         cplx_t<T>* __restrict__ M) {
  extern __shared__ __align__(16) unsigned char smem[];
  cplx_t<T>* As = (cplx_t<T>*)smem;      // [2][kBK][kBM]
  cplx_t<T>* Bs = As + 2 * kBK * kBM;    // [2][kBK][kBN]
  const int L = tl.L;
  const int64_t t = blockIdx.x;
  int i = 0;
  while (t >= tl.start[i + 1]) ++i;      // uniform walk over <= L + 1 entries (constant bank)
  const int l = L - i, w = 2 * l + 1, ct = col_tiles(l);
  const int64_t local = t - tl.start[i];
  const int64_t rt = local / ct;
  const int c0 = (int)(local - rt * ct) * kBN;
  const int64_t rho0 = rt * kBM, nrows = B * (l + 1);
  const int ncf = ncoef(Lmax);
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  // staging assignments: A row ar, shells ak..ak+3; B column bc, shells bk..bk+3
  const int ar = tid >> 2, ak = (tid & 3) * 4, bc = tid & 63, bk = (tid >> 6) * 4;
  const int64_t rho = rho0 + ar;
  const cplx_t<T>* Frow = nullptr;
  if (rho < nrows) {
    const int64_t p = rho / (l + 1);
    const int m = (int)(rho - p * (l + 1));
    Frow = F + p * (int64_t)ncf * R + (int64_t)(lm_index(l, 0) + m) * R;
  }
  const int n = c0 + bc - l;
  const cplx_t<T>* Hrow = (c0 + bc < w) ? H + (int64_t)lm_index(l, abs(n)) * R : nullptr;
  const cplx_t<T> zero = mk<T>(T(0), T(0));
  cplx_t<T> ra[4], rb[4];
  auto fetch = [&](int r0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + ak + j;
      ra[j] = (Frow && r < R) ? Frow[r] : zero;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + bk + j;
      cplx_t<T> v = zero;
      if (Hrow && r < R) {
        const T rr = (T)r + T(0.5), wr = rr * rr;
        const cplx_t<T> h = Hrow[r];
        if (n >= 0) v = mk<T>(wr * h.x, -wr * h.y);                                  // w conj(h_{l,n})
        else v = (n & 1) ? mk<T>(-wr * h.x, -wr * h.y) : mk<T>(wr * h.x, wr * h.y);  // w (-1)^n h_{l,|n|}
      }
      rb[j] = v;
    }
  };
  auto stash = [&](int buf) {
    cplx_t<T>* a = As + buf * kBK * kBM;
    cplx_t<T>* b = Bs + buf * kBK * kBN;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      a[(ak + j) * kBM + ar] = ra[j];
      b[(bk + j) * kBN + bc] = rb[j];
    }
  };
  T accr[4][4], acci[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) accr[u][v] = acci[u][v] = T(0);
  const int nch = (R + kBK - 1) / kBK;
  fetch(0);
  stash(0);
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) fetch((c + 1) * kBK);  // global loads of chunk c + 1 in flight during the FMAs of chunk c
    const cplx_t<T>* a = As + buf * kBK * kBM + ty * 4;
    const cplx_t<T>* b = Bs + buf * kBK * kBN + tx;
#pragma unroll
    for (int k = 0; k < kBK; ++k) {
      cplx_t<T> av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = a[k * kBM + u];
#pragma unroll
      for (int v = 0; v < 4; ++v) bv[v] = b[k * kBN + 16 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          accr[u][v] = fma(av[u].x, bv[v].x, fma(-av[u].y, bv[v].y, accr[u][v]));
          acci[u][v] = fma(av[u].x, bv[v].y, fma(av[u].y, bv[v].x, acci[u][v]));
        }
    }
    if (c + 1 < nch) stash(buf ^ 1);
    __syncthreads();
  }
  const int64_t hs = half_size(L), ho = half_offset(l);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t r = rho0 + ty * 4 + u;
    if (r >= nrows) continue;
    const int64_t p = r / (l + 1);
    const int m = (int)(r - p * (l + 1));
    cplx_t<T>* Mo = M + p * hs + ho + (int64_t)m * w;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int col = c0 + tx + 16 * v;
      if (col < w) Mo[col] = mk<T>(accr[u][v], acci[u][v]);
    }
  }
}

}  // namespace

template <typename T>
cudaError_t launch_corr_coeffs(const cplx_t<T>* F, const cplx_t<T>* H, int64_t B, int L, int Lmax, int R,
                               cplx_t<T>* M, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  if (L > kMaxL) return cudaErrorInvalidValue;
  CorrTiles tl;
  tl.L = L;
  tl.start[0] = 0;
  for (int i = 0; i <= L; ++i) {
    const int l = L - i;
    tl.start[i + 1] = tl.start[i] + (B * (l + 1) + kBM - 1) / kBM * col_tiles(l);
  }
  const size_t bytes = sizeof(cplx_t<T>) * 2 * kBK * (kBM + kBN);
  cudaError_t e = cudaFuncSetAttribute(k_corr_tiled<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  k_corr_tiled<T><<<(unsigned)tl.start[L + 1], kThreads, bytes, s>>>(F, H, B, Lmax, R, tl, M);
  return cudaGetLastError();
}

template cudaError_t launch_corr_coeffs<float>(const float2*, const float2*, int64_t, int, int, int, float2*,
                                               cudaStream_t);
template cudaError_t launch_corr_coeffs<double>(const double2*, const double2*, int64_t, int, int, int, double2*,
                                                cudaStream_t);

}  // namespace matcha
