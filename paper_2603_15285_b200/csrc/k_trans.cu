// k_trans.cu -- stage 5: the translation update of the rotation/translation alternation.
//
// PAPER.md App. C: for fixed g, the best translation is found "on a fine grid by evaluating
// the cross-correlation with 3D FFT", restricted to a local window (remark iv), with
// subpixel refinement (remark iii).  Readings C17 (t in the particle frame, f ~ S_t(g o h)) and
// C18 (circular correlation, window [-W,W]^3, ties -> lowest window index z-major, parabolic subpixel
// per axis clamped to 1/2, trilinear rotation of the reference, zero outside):
//   rho(x) = h(R^T (x - c) + c),   c(t) = sum_x f(x) rho((x - t) mod N) = IFFT(F^ conj(rho^))(t) / N^3.
//
// B200 mapping: the rotated references of a chunk are produced by one gather kernel (the reference is
// shared by every particle and stays L2-resident), the 3-D transforms are batched cuFFT R2C/C2R plans
// (library, like cuBLAS), the cross spectrum is an in-place elementwise kernel, and the windowed argmax +
// subpixel fit is one CTA per particle with a deterministic (value desc, index asc) block reduction.
#include "common.cuh"

namespace matcha {

namespace {

template <typename T> __device__ __forceinline__ void rot_matrix(const T* e, double* R) {
  const double a = (double)e[0], b = (double)e[1], g = (double)e[2];
  double sa, ca, sb, cb, sg, cg;
  sincos(a, &sa, &ca);
  sincos(b, &sb, &cb);
  sincos(g, &sg, &cg);
  // r_z(a) r_y(b) r_z(g)  (Eq. 3)
  R[0] = ca * cb * cg - sa * sg;
  R[1] = -ca * cb * sg - sa * cg;
  R[2] = ca * sb;
  R[3] = sa * cb * cg + ca * sg;
  R[4] = -sa * cb * sg + ca * cg;
  R[5] = sa * sb;
  R[6] = -sb * cg;
  R[7] = sb * sg;
  R[8] = cb;
}

template <typename T>
__device__ __forceinline__ T trilinear_g(const float* __restrict__ v, int N, T px, T py, T pz) {
  const T fx0 = floor(px), fy0 = floor(py), fz0 = floor(pz);
  const int x0 = (int)fx0, y0 = (int)fy0, z0 = (int)fz0;
  const T fx = px - fx0, fy = py - fy0, fz = pz - fz0;
  T c[2][2][2];
#pragma unroll
  for (int dz = 0; dz < 2; ++dz)
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const int x = x0 + dx, y = y0 + dy, z = z0 + dz;
        const bool in = (unsigned)x < (unsigned)N && (unsigned)y < (unsigned)N && (unsigned)z < (unsigned)N;
        c[dz][dy][dx] = in ? (T)__ldg(v + ((size_t)z * N + y) * N + x) : T(0);
      }
  const T c00 = fma(fx, c[0][0][1] - c[0][0][0], c[0][0][0]);
  const T c01 = fma(fx, c[0][1][1] - c[0][1][0], c[0][1][0]);
  const T c10 = fma(fx, c[1][0][1] - c[1][0][0], c[1][0][0]);
  const T c11 = fma(fx, c[1][1][1] - c[1][1][0], c[1][1][0]);
  const T c0 = fma(fy, c01 - c00, c00);
  const T c1 = fma(fy, c11 - c10, c10);
  return fma(fz, c1 - c0, c0);
}

// rho_p(x) = h(R_p^T (x - c) + c) for particles p < nb; euler rows at stride estride
template <typename T>
__global__ void __launch_bounds__(256) k_rotate_ref(const float* __restrict__ ref, int N, const T* __restrict__ euler,
                                                    int estride, T* __restrict__ rho) {
  __shared__ double Rm[9];
  const int64_t p = blockIdx.y;
  if (threadIdx.x == 0) rot_matrix<T>(euler + p * estride, Rm);
  __syncthreads();
  const int64_t n3 = (int64_t)N * N * N;
  const T c = T(0.5) * (T)(N - 1);
  const T r0 = (T)Rm[0], r1 = (T)Rm[1], r2 = (T)Rm[2], r3 = (T)Rm[3], r4 = (T)Rm[4], r5 = (T)Rm[5], r6 = (T)Rm[6],
          r7 = (T)Rm[7], r8 = (T)Rm[8];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n3; v += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(v % N), y = (int)((v / N) % N), z = (int)(v / ((int64_t)N * N));
    const T vx = (T)x - c, vy = (T)y - c, vz = (T)z - c;
    const T qx = fma(r0, vx, fma(r3, vy, r6 * vz)) + c;  // R^T v
    const T qy = fma(r1, vx, fma(r4, vy, r7 * vz)) + c;
    const T qz = fma(r2, vx, fma(r5, vy, r8 * vz)) + c;
    rho[p * n3 + v] = trilinear_g<T>(ref, N, qx, qy, qz);
  }
}

template <typename T>
__global__ void k_to_real(const float* __restrict__ in, T* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (T)in[i];
}

// X <- F^ . conj(X), elementwise
template <typename T>
__global__ void k_cross_spectrum(const cplx_t<T>* __restrict__ F, cplx_t<T>* __restrict__ X, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const cplx_t<T> f = F[i], x = X[i];
    X[i] = mk<T>(f.x * x.x + f.y * x.y, f.y * x.x - f.x * x.y);
  }
}

template <typename T> __device__ __forceinline__ bool better(T v1, int i1, T v2, int i2) {
  return v1 > v2 || (v1 == v2 && i1 < i2);
}

// windowed argmax (ties -> lowest window index, z-major) + per-axis parabolic subpixel; corr = N^3 c(t)
template <typename T>
__global__ void __launch_bounds__(256) k_window_peak(const T* __restrict__ corr, int N, int W, T* shifts, int sstride,
                                                     T* peak) {
  __shared__ T sv[8];
  __shared__ int si[8];
  const int64_t p = blockIdx.x;
  const T* cp = corr + p * (int64_t)N * N * N;
  const int w = 2 * W + 1, nw = w * w * w;
  auto at = [&](int tx, int ty, int tz) {
    const int x = ((tx % N) + N) % N, y = ((ty % N) + N) % N, z = ((tz % N) + N) % N;
    return cp[((size_t)z * N + y) * N + x];
  };
  T bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int t = threadIdx.x; t < nw; t += blockDim.x) {
    const int tx = t % w - W, ty = (t / w) % w - W, tz = t / (w * w) - W;
    const T v = at(tx, ty, tz);
    if (better(v, t, bv, bi)) {
      bv = v;
      bi = t;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T v2 = __shfl_xor_sync(0xffffffffu, bv, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(v2, i2, bv, bi)) {
      bv = v2;
      bi = i2;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sv[warp] = bv;
    si[warp] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (better(sv[k], si[k], bv, bi)) {
        bv = sv[k];
        bi = si[k];
      }
    const int t[3] = {bi % w - W, (bi / w) % w - W, bi / (w * w) - W};
    const T c0 = bv;
    for (int ax = 0; ax < 3; ++ax) {
      int tm[3] = {t[0], t[1], t[2]}, tp[3] = {t[0], t[1], t[2]};
      tm[ax] -= 1;
      tp[ax] += 1;
      const T cm = at(tm[0], tm[1], tm[2]), cpl = at(tp[0], tp[1], tp[2]);
      const T den = cm - T(2) * c0 + cpl;
      T dl = T(0);
      if (den < T(0)) dl = fmin(T(0.5), fmax(T(-0.5), (cm - cpl) / (T(2) * den)));
      shifts[p * sstride + ax] = (T)t[ax] + dl;
    }
    if (peak) peak[p] = c0 / ((T)N * N * N);
  }
}

}  // namespace

template <typename T>
cudaError_t launch_rotate_ref(const float* ref, int N, const T* euler, int estride, int64_t nb, T* rho,
                              cudaStream_t s) {
  if (nb == 0) return cudaSuccess;
  const int64_t n3 = (int64_t)N * N * N;
  dim3 grid((unsigned)std::min<int64_t>((n3 + 255) / 256, 4096), (unsigned)nb);
  k_rotate_ref<T><<<grid, 256, 0, s>>>(ref, N, euler, estride, rho);
  return cudaGetLastError();
}

template <typename T> cudaError_t launch_to_real(const float* in, T* out, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_to_real<T><<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s>>>(in, out, n);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_cross_spectrum(const cplx_t<T>* F, cplx_t<T>* X, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_cross_spectrum<T><<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s>>>(F, X, n);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_window_peak(const T* corr, int N, int W, int64_t nb, T* shifts, int sstride, T* peak,
                               cudaStream_t s) {
  if (nb == 0) return cudaSuccess;
  k_window_peak<T><<<(unsigned)nb, 256, 0, s>>>(corr, N, W, shifts, sstride, peak);
  return cudaGetLastError();
}

template cudaError_t launch_rotate_ref<float>(const float*, int, const float*, int, int64_t, float*, cudaStream_t);
template cudaError_t launch_rotate_ref<double>(const float*, int, const double*, int, int64_t, double*, cudaStream_t);
template cudaError_t launch_to_real<float>(const float*, float*, int64_t, cudaStream_t);
template cudaError_t launch_to_real<double>(const float*, double*, int64_t, cudaStream_t);
template cudaError_t launch_cross_spectrum<float>(const float2*, float2*, int64_t, cudaStream_t);
template cudaError_t launch_cross_spectrum<double>(const double2*, double2*, int64_t, cudaStream_t);
template cudaError_t launch_window_peak<float>(const float*, int, int, int64_t, float*, int, float*, cudaStream_t);
template cudaError_t launch_window_peak<double>(const double*, int, int, int64_t, double*, int, double*,
                                                cudaStream_t);

}  // namespace matcha
