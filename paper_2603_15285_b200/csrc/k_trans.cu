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

// rho_p(x) = h(R_p^T (x - c) + c) for particles p < nb; euler rows at stride estride.
// One CTA per (8^3 output tile, particle): the tile's source region (the axis-aligned box around the rotated
// cube, <= 16^3 voxels incl. the trilinear +1) is staged in shared memory by row loads from the L2-resident
// reference, then every voxel gathers its 8 corners from shared memory.  (A direct gather from L2 touches a
// separate 32-byte sector for nearly every lane of a rotated row: ~0.25 voxel per cycle per SM.)  Out-of-volume
// corners are staged as 0, so the arithmetic is exactly trilinear_g's.  N is a multiple of 8 (matcha_create).
constexpr int kRotTile = 8, kRotBox = 16, kRotCtas = 96;
template <typename T>
__global__ void __launch_bounds__(256) k_rotate_ref(const float* __restrict__ ref, int N, const T* __restrict__ euler,
                                                    int estride, T* __restrict__ rho) {
  __shared__ double Rm[9];
  __shared__ float box[kRotBox * kRotBox * kRotBox];
  const int64_t p = blockIdx.y;
  const int nt = N / kRotTile;
  const T c = T(0.5) * (T)(N - 1);
  if (threadIdx.x == 0) rot_matrix<T>(euler + p * estride, Rm);
  __syncthreads();
  const T r0 = (T)Rm[0], r1 = (T)Rm[1], r2 = (T)Rm[2], r3 = (T)Rm[3], r4 = (T)Rm[4], r5 = (T)Rm[5], r6 = (T)Rm[6],
          r7 = (T)Rm[7], r8 = (T)Rm[8];
  // half extent of the image of a tile (cube of edge kRotTile-1 voxels) along each source axis
  const T hE = T(0.5) * (T)(kRotTile - 1);
  const T ex = hE * (fabs(r0) + fabs(r3) + fabs(r6)), ey = hE * (fabs(r1) + fabs(r4) + fabs(r7)),
          ez = hE * (fabs(r2) + fabs(r5) + fabs(r8));
  T* out = rho + p * (int64_t)N * N * N;
  // tile coordinates advanced by gridDim.x with carries (no per-tile integer division)
  int tx = blockIdx.x % nt, ty = (blockIdx.x / nt) % nt, tz = blockIdx.x / (nt * nt);
  const int sx = gridDim.x % nt, sy = (gridDim.x / nt) % nt, sz = gridDim.x / (nt * nt);
  for (; tz < nt; tx += sx, ty += sy, tz += sz) {
    if (tx >= nt) {
      tx -= nt;
      ++ty;
    }
    if (ty >= nt) {
      ty -= nt;
      ++tz;
    }
    if (tz >= nt) break;
    // source box: image centre +- extent (+ margin against rounding), corners floor(q) .. floor(q) + 1
    const T vx = (T)tx * kRotTile + hE - c, vy = (T)ty * kRotTile + hE - c, vz = (T)tz * kRotTile + hE - c;
    const T qcx = fma(r0, vx, fma(r3, vy, r6 * vz)) + c, qcy = fma(r1, vx, fma(r4, vy, r7 * vz)) + c,
            qcz = fma(r2, vx, fma(r5, vy, r8 * vz)) + c;
    const int ox = (int)floor(qcx - ex - T(1e-3)), oy = (int)floor(qcy - ey - T(1e-3)),
              oz = (int)floor(qcz - ez - T(1e-3));
    const int dx = (int)floor(qcx + ex + T(1e-3)) + 2 - ox, dy = (int)floor(qcy + ey + T(1e-3)) + 2 - oy,
              dz = (int)floor(qcz + ez + T(1e-3)) + 2 - oz;
    // the box always fits: each extent is 2e + 3 + 0.002 <= 7 sqrt(3) + 3.002 < 16 voxels at kRotTile = 8, and by
    // construction every voxel's corners floor(q) .. floor(q) + 1 lie inside it (static_assert below)
    static_assert(kRotTile == 8 && kRotBox == 16, "box bound derived for 8^3 tiles");
    __syncthreads();  // previous tile's gathers are done with the box
    {
      // one (y, x) slice of the box per pass: thread -> (iy, ix) = (tid / 16, tid % 16), no index division
      const int ix = threadIdx.x & (kRotBox - 1), iy = threadIdx.x / kRotBox;
      const int x = ox + ix, y = oy + iy;
      const bool inxy = ix < dx && iy < dy;
      const bool vxy = (unsigned)x < (unsigned)N && (unsigned)y < (unsigned)N;
      if (inxy && threadIdx.x < kRotBox * kRotBox) {
        float* dst = box + iy * kRotBox + ix;
        // all of the column's loads in flight before the first store (a load -> store loop serialised ~dz L2
        // latencies per tile); 32-bit plane offsets (N^3 < 2^31), one pointer per column
        const int NN = N * N;
        const float* src = ref + (vxy ? y * N + x : 0);
        float col[kRotBox];
#pragma unroll
        for (int iz = 0; iz < kRotBox; ++iz) {
          const int z = oz + iz;
          col[iz] = (iz < dz && vxy && (unsigned)z < (unsigned)N) ? __ldg(src + z * NN) : 0.f;
        }
#pragma unroll
        for (int iz = 0; iz < kRotBox; ++iz)
          if (iz < dz) dst[iz * kRotBox * kRotBox] = col[iz];
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kRotTile * kRotTile * kRotTile; i += blockDim.x) {
      const int x = tx * kRotTile + (i % kRotTile), y = ty * kRotTile + (i / kRotTile) % kRotTile,
                z = tz * kRotTile + i / (kRotTile * kRotTile);
      const T ux = (T)x - c, uy = (T)y - c, uz = (T)z - c;
      const T qx = fma(r0, ux, fma(r3, uy, r6 * uz)) + c;  // R^T v
      const T qy = fma(r1, ux, fma(r4, uy, r7 * uz)) + c;
      const T qz = fma(r2, ux, fma(r5, uy, r8 * uz)) + c;
      const T fx0 = floor(qx), fy0 = floor(qy), fz0 = floor(qz);
      const int bx = (int)fx0 - ox, by = (int)fy0 - oy, bz = (int)fz0 - oz;
      const T fx = qx - fx0, fy = qy - fy0, fz = qz - fz0;
      const float* b0 = box + (bz * kRotBox + by) * kRotBox + bx;
      const T c000 = b0[0], c001 = b0[1], c010 = b0[kRotBox], c011 = b0[kRotBox + 1];
      const T c100 = b0[kRotBox * kRotBox], c101 = b0[kRotBox * kRotBox + 1];
      const T c110 = b0[kRotBox * kRotBox + kRotBox], c111 = b0[kRotBox * kRotBox + kRotBox + 1];
      const T c00 = fma(fx, c001 - c000, c000);
      const T c01 = fma(fx, c011 - c010, c010);
      const T c10 = fma(fx, c101 - c100, c100);
      const T c11 = fma(fx, c111 - c110, c110);
      const T c0 = fma(fy, c01 - c00, c00);
      const T c1 = fma(fy, c11 - c10, c10);
      const T val = fma(fz, c1 - c0, c0);
      out[(z * N + y) * N + x] = val;
    }
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

// ---- windowed correlation by a pruned inverse DFT (replaces the cross spectrum + full C2R + window read) --------
// Only c(t) for t in the window [-W-1, W+1]^3 (the argmax window plus the subpixel neighbours) is needed, so the
// inverse transform of X = F^ conj(rho^) is evaluated directly on those w' = 2W+3 points per axis, separably:
//   Y1[kz][ky][a]  = sum_{kx=0}^{N/2} w_kx X[kz][ky][kx] e^{+2 pi i kx tx_a / N}   (w_kx = 1 at kx = 0, N/2, else 2)
//   Y2[kz][b][a]   = sum_ky Y1[kz][ky][a] e^{+2 pi i ky ty_b / N}
//   cw[c][b][a]    = Re sum_kz Y2[kz][b][a] e^{+2 pi i kz tz_c / N}  = N^3 c(t)  (the unnormalised C2R value)
// X is Hermitian (F^, rho^ are spectra of real volumes), so the half-spectrum sum with weights w_kx and Re is exact.
// The per-(particle, kz) kernel forms X in shared memory from coalesced F^/rho^ plane loads (X is never stored).

template <typename T> __device__ __forceinline__ cplx_t<T> cmul(cplx_t<T> a, cplx_t<T> b) {
  return mk<T>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

template <typename T>
__device__ __forceinline__ void build_twiddles(cplx_t<T>* tw, int N) {
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    double sn, cs;
    sincospi(2.0 * j / N, &sn, &cs);  // e^{+2 pi i j / N}
    tw[j] = mk<T>((T)cs, (T)sn);
  }
}

// grid (N, nb): block (kz, p) -> Y2[p][kz][w'][w']
template <typename T>
__global__ void __launch_bounds__(512) k_window_xy(const cplx_t<T>* __restrict__ Fh, const cplx_t<T>* __restrict__ Rh,
                                                   int N, int W, cplx_t<T>* __restrict__ Y2) {
  extern __shared__ unsigned char smem_raw[];
  const int H = N / 2 + 1, wp = 2 * W + 3;
  cplx_t<T>* tw = reinterpret_cast<cplx_t<T>*>(smem_raw);  // [N][wp]: e^{+2 pi i k t_a / N}, t_a = a - (W+1)
  cplx_t<T>* X = tw + N * wp;                              // [N][H]
  cplx_t<T>* Y1 = X + N * H;                               // [N][wp]
  cplx_t<T>* base = Y1 + N * wp;                           // [N]: e^{+2 pi i j / N}
  const int kz = blockIdx.x;
  const int64_t p = blockIdx.y;
  const int64_t plane = ((int64_t)p * N + kz) * N * H;
  build_twiddles<T>(base, N);
  __syncthreads();
  for (int i = threadIdx.x; i < N * wp; i += blockDim.x) {
    const int k = i / wp, t = i - k * wp - (W + 1);
    tw[i] = base[(((k * t) % N) + N) % N];
  }
  // four elements per thread per pass, all eight loads issued before the first use (the loads' latency, not the
  // arithmetic, paced the one-element loop)
  constexpr int kU = 4;
  for (int i0 = threadIdx.x; i0 < N * H; i0 += kU * blockDim.x) {
    cplx_t<T> f[kU], r[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < N * H) {
        f[u] = Fh[plane + i];
        r[u] = Rh[plane + i];
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < N * H) {
        const int kx = i % H;
        const T wk = (kx == 0 || 2 * kx == N) ? T(1) : T(2);
        X[i] = mk<T>(wk * (f[u].x * r[u].x + f[u].y * r[u].y), wk * (f[u].y * r[u].x - f[u].x * r[u].y));  // w F^ conj(rho^)
      }
    }
  }
  __syncthreads();
  for (int o = threadIdx.x; o < N * wp; o += blockDim.x) {
    const int ky = o / wp, a = o - ky * wp;
    const cplx_t<T>* xr = X + ky * H;
    T ar = T(0), ai = T(0);
    for (int kx = 0; kx < H; ++kx) {
      const cplx_t<T> x = xr[kx], t = tw[kx * wp + a];
      ar = fma(x.x, t.x, fma(-x.y, t.y, ar));
      ai = fma(x.x, t.y, fma(x.y, t.x, ai));
    }
    Y1[o] = mk<T>(ar, ai);
  }
  __syncthreads();
  for (int o = threadIdx.x; o < wp * wp; o += blockDim.x) {
    const int b = o / wp, a = o - b * wp;
    T ar = T(0), ai = T(0);
    for (int ky = 0; ky < N; ++ky) {
      const cplx_t<T> y = Y1[ky * wp + a], t = tw[ky * wp + b];
      ar = fma(y.x, t.x, fma(-y.y, t.y, ar));
      ai = fma(y.x, t.y, fma(y.y, t.x, ai));
    }
    Y2[((int64_t)p * N + kz) * wp * wp + o] = mk<T>(ar, ai);
  }
}

// grid nb: the z pass into cw[p][w'^3] (global scratch), then the windowed argmax (ties -> lowest window index,
// z-major) and the per-axis parabolic subpixel (reading C18), as k_window_peak but on the pruned window
template <typename T>
__global__ void __launch_bounds__(256) k_window_z_peak(const cplx_t<T>* __restrict__ Y2, int N, int W,
                                                       T* __restrict__ cw_all, T* shifts, int sstride, T* peak) {
  __shared__ cplx_t<T> tw[512];
  __shared__ T sv[8];
  __shared__ int si[8];
  const int64_t p = blockIdx.x;
  const int wp = 2 * W + 3, w = 2 * W + 1, wp2 = wp * wp;
  build_twiddles<T>(tw, N);
  __syncthreads();
  const cplx_t<T>* y2 = Y2 + p * (int64_t)N * wp2;
  T* cw = cw_all + p * (int64_t)wp2 * wp;
  for (int o = threadIdx.x; o < wp2 * wp; o += blockDim.x) {
    const int c = o / wp2, ba = o - c * wp2;
    const int tz = c - (W + 1);
    const int step = ((tz % N) + N) % N;
    T acc = T(0);
    int idx = 0;
    for (int kz = 0; kz < N; ++kz) {
      const cplx_t<T> y = y2[(int64_t)kz * wp2 + ba], t = tw[idx];
      acc = fma(y.x, t.x, fma(-y.y, t.y, acc));
      idx += step;
      if (idx >= N) idx -= N;
    }
    cw[o] = acc;
  }
  __syncthreads();
  auto at = [&](int tx, int ty, int tz) { return cw[((tz + W + 1) * wp + (ty + W + 1)) * wp + (tx + W + 1)]; };
  const int nw = w * w * w;
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
  (void)n3;
  if (N % kRotTile) return cudaErrorInvalidValue;
  const int nt = N / kRotTile;
  k_rotate_ref<T><<<dim3((unsigned)std::min(nt * nt * nt, kRotCtas), (unsigned)nb), 256, 0, s>>>(ref, N, euler,
                                                                                                  estride, rho);
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

size_t window_scratch_reals(int N, int W) {
  const int64_t wp = 2 * W + 3;
  return (size_t)(2 * (int64_t)N * wp * wp + wp * wp * wp);
}

// Y2 and the c window of particle p live in scratch + p * window_scratch_reals(N, W) reals
template <typename T>
cudaError_t launch_window_pruned(const cplx_t<T>* Fh, const cplx_t<T>* Rh, int N, int W, int64_t nb, T* scratch,
                                 T* shifts, int sstride, T* peak, cudaStream_t s) {
  if (nb == 0) return cudaSuccess;
  if (N > 512 || 2 * W + 3 > N) return cudaErrorInvalidValue;
  const int H = N / 2 + 1, wp = 2 * W + 3;
  const size_t smem = sizeof(cplx_t<T>) * ((size_t)N * wp + (size_t)N * H + (size_t)N * wp + (size_t)N);
  cudaError_t e = cudaFuncSetAttribute(k_window_xy<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // Y2 [nb][N][wp][wp] complex at the front of the scratch, the c windows [nb][wp^3] behind it
  cplx_t<T>* Y2 = reinterpret_cast<cplx_t<T>*>(scratch);
  T* cw = scratch + 2 * nb * (int64_t)N * wp * wp;
  k_window_xy<T><<<dim3((unsigned)N, (unsigned)nb), 512, smem, s>>>(Fh, Rh, N, W, Y2);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_window_z_peak<T><<<(unsigned)nb, 256, 0, s>>>(Y2, N, W, cw, shifts, sstride, peak);
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
template cudaError_t launch_window_pruned<float>(const float2*, const float2*, int, int, int64_t, float*, float*, int,
                                                 float*, cudaStream_t);
template cudaError_t launch_window_pruned<double>(const double2*, const double2*, int, int, int64_t, double*, double*,
                                                  int, double*, cudaStream_t);

}  // namespace matcha
