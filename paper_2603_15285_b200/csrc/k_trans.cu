// k_trans.cu -- stage 5: the translation update of the rotation/translation alternation.
//
// PAPER.md App. C: for fixed g, the best translation is found "on a fine grid by evaluating
// the cross-correlation with 3D FFT", restricted to a local window (remark iv), with
// subpixel refinement (remark iii).  Readings C17 (t in the particle frame, f ~ S_t(g o h)) and
// C18 (circular correlation, window [-W,W]^3, ties -> lowest window index z-major, parabolic subpixel
// per axis clamped to 1/2, trilinear rotation of the reference, zero outside):
//   rho(x) = h(R^T (x - c) + c),   c(t) = sum_x f(x) rho((x - t) mod N) = IFFT(F^ conj(rho^))(t) / N^3.
//
// B200 mapping (no FFT library): the inverse transform is needed only on the window, and its kz part at integer
// tz is a circular correlation ALONG z of the 2-D (x, y) plane spectra, so no z transform is ever done:
//   5a k_plane_r2c   2-D R2C of every z-plane (hand-written mixed-radix Stockham FFTs in shared memory, two real
//                    rows per complex line): f~ of the particles once per chunk, rho~ of the rotated references
//                    (k_rotate_ref, the reference is L2-resident) every alternation;
//   5b k_zcorr       Y1(kx, ky, tz) = sum_z f~(kx, ky, z + tz) conj(rho~(kx, ky, z)) for the w' = 2W + 3 window tz;
//   5c k_window_xy   the (x, y) inverse onto the window (tx, ty) from Y1, Hermitian half spectrum, Re;
//   5d k_window_peak the windowed argmax and the per-axis parabolic subpixel fit (deterministic block reduction).
// N^2 c(t) = Re sum_{kx,ky} w_kx e^{2 pi i (kx tx + ky ty)/N} Y1(kx, ky, tz)   (exact: Parseval in x, y + the z shift).
#include <algorithm>

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
__global__ void __launch_bounds__(256) k_rotate_ref(const float* __restrict__ refs, int N, const T* __restrict__ euler,
                                                    int estride, const int* __restrict__ tsel, T* __restrict__ rho) {
  __shared__ double Rm[9];
  __shared__ float box[kRotBox * kRotBox * kRotBox];
  const int64_t p = blockIdx.y;
  // multi-template alignment: particle p's translation uses its selected template
  const float* ref = refs + (tsel ? (int64_t)tsel[p] * N * N * N : 0);
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

template <typename T> __device__ __forceinline__ bool better(T v1, int i1, T v2, int i2) {
  return v1 > v2 || (v1 == v2 && i1 < i2);
}

template <typename T> __device__ __forceinline__ cplx_t<T> cmul(cplx_t<T> a, cplx_t<T> b) {
  return mk<T>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <typename T> __device__ __forceinline__ cplx_t<T> cadd(cplx_t<T> a, cplx_t<T> b) {
  return mk<T>(a.x + b.x, a.y + b.y);
}
template <typename T> __device__ __forceinline__ cplx_t<T> csub(cplx_t<T> a, cplx_t<T> b) {
  return mk<T>(a.x - b.x, a.y - b.y);
}
// a * (-i)
template <typename T> __device__ __forceinline__ cplx_t<T> cmi(cplx_t<T> a) { return mk<T>(a.y, -a.x); }

// tw[m] = e^{sign 2 pi i m / n}, m < n (FP64 sincospi, cast)
template <typename T> __device__ __forceinline__ void build_roots(cplx_t<T>* tw, int n, int sign) {
  for (int m = threadIdx.x; m < n; m += blockDim.x) {
    double sn, cs;
    sincospi(2.0 * m / n, &sn, &cs);
    tw[m] = mk<T>((T)cs, (T)(sign * sn));
  }
}

// ---- batched 1-D FFTs in shared memory (mixed-radix Stockham autosort, forward e^{-2 pi i k n / N}) ----------
// nl independent lines of length n = fr.n, line l at a[l * n + i].  Stage s (radix R = fr.rad[s], Ns = product of the
// previous radices) combines R sub-transforms of length Ns: butterfly j (< n / R) reads a[j + r n / R], twiddles input
// r by e^{-2 pi i r (j mod Ns) / (Ns R)} = tw[r (j mod Ns) n / (Ns R)], applies the R-point DFT and writes
// b[(j - j mod Ns) R + j mod Ns + q Ns].  Radix 4, 2, 3 are specialised; any other prime factor (N is a multiple of 8,
// so only N with factors 5, 7, 11, ... reach it) runs the direct R-point DFT.  All threads of the CTA must call it;
// it ends with __syncthreads() after every stage and returns the buffer that holds the result (a or b).
template <typename T>
__device__ cplx_t<T>* stockham(cplx_t<T>* a, cplx_t<T>* b, int nl, const FftRadix& fr, const cplx_t<T>* __restrict__ tw) {
  const int n = fr.n;
  int Ns = 1;
  for (int s = 0; s < fr.nst; ++s) {
    const int R = fr.rad[s], nb = n / R, ts = n / (Ns * R);
    for (int t = threadIdx.x; t < nl * nb; t += blockDim.x) {
      const int l = t / nb, j = t - l * nb, k = j % Ns;
      const cplx_t<T>* in = a + l * n + j;
      cplx_t<T>* out = b + l * n + (j - k) * R + k;
      if (R == 4) {
        const cplx_t<T> v0 = in[0], v1 = cmul<T>(in[nb], tw[k * ts]), v2 = cmul<T>(in[2 * nb], tw[2 * k * ts]),
                        v3 = cmul<T>(in[3 * nb], tw[3 * k * ts]);
        const cplx_t<T> s02 = cadd<T>(v0, v2), d02 = csub<T>(v0, v2), s13 = cadd<T>(v1, v3), d13 = cmi<T>(csub<T>(v1, v3));
        out[0] = cadd<T>(s02, s13);
        out[Ns] = cadd<T>(d02, d13);
        out[2 * Ns] = csub<T>(s02, s13);
        out[3 * Ns] = csub<T>(d02, d13);
      } else if (R == 2) {
        const cplx_t<T> v0 = in[0], v1 = cmul<T>(in[nb], tw[k * ts]);
        out[0] = cadd<T>(v0, v1);
        out[Ns] = csub<T>(v0, v1);
      } else if (R == 3) {
        const cplx_t<T> v0 = in[0], v1 = cmul<T>(in[nb], tw[k * ts]), v2 = cmul<T>(in[2 * nb], tw[2 * k * ts]);
        const T h = T(0.86602540378443864676);  // sin(2 pi / 3)
        const cplx_t<T> sm = cadd<T>(v1, v2), df = csub<T>(v1, v2);
        const cplx_t<T> m = mk<T>(v0.x - T(0.5) * sm.x, v0.y - T(0.5) * sm.y);
        out[0] = cadd<T>(v0, sm);
        out[Ns] = mk<T>(m.x + h * df.y, m.y - h * df.x);      // m - i h df
        out[2 * Ns] = mk<T>(m.x - h * df.y, m.y + h * df.x);  // m + i h df
      } else {
        const int nR = n / R;
        for (int q = 0; q < R; ++q) {
          cplx_t<T> acc = mk<T>(T(0), T(0));
          for (int r = 0; r < R; ++r) {
            const cplx_t<T> v = r ? cmul<T>(in[r * nb], tw[r * k * ts]) : in[0];
            acc = cadd<T>(acc, cmul<T>(v, tw[((r * q) % R) * nR]));
          }
          out[q * Ns] = acc;
        }
      }
    }
    __syncthreads();
    cplx_t<T>* x = a;
    a = b;
    b = x;
    Ns *= R;
  }
  return a;
}

// ---- stage 5a: 2-D R2C transform of every z-plane of a real volume -----------------------------------------------
//   U~[p][z][ky][kx] = sum_{y,x} u_p(x, y, z) e^{-2 pi i (kx x + ky y) / N},   kx in [0, N/2]
// One CTA per (plane, particle).  x pass: rows 2y', 2y'+1 packed as one complex line a + i b, transformed together,
// then unpacked, A(k) = (Z(k) + conj Z(N-k)) / 2, B(k) = (Z(k) - conj Z(N-k)) / (2i); the half rows land in the plane
// buffer P[N][H].  y pass: columns of P in chunks of cwl lines, transformed back into P.  P is written out linearly.
// Used for the particles (once per chunk: f~) and for the rotated references (every alternation: rho~).
template <typename T, typename Tin>
__global__ void __launch_bounds__(256) k_plane_r2c(const Tin* __restrict__ vol, const __grid_constant__ FftRadix fr,
                                                   int cwl,
                                                   cplx_t<T>* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = fr.n, H = N / 2 + 1;
  cplx_t<T>* tw = reinterpret_cast<cplx_t<T>*>(smem_raw);
  cplx_t<T>* P = tw + N;
  cplx_t<T>* S0 = P + N * H;
  cplx_t<T>* S1 = S0 + cwl * N;
  const int z = blockIdx.x;
  const int64_t p = blockIdx.y;
  const Tin* u = vol + (p * N + z) * (int64_t)N * N;
  build_roots<T>(tw, N, -1);
  for (int y0 = 0; y0 < N / 2; y0 += cwl) {
    const int nl = min(cwl, N / 2 - y0);
    for (int i = threadIdx.x; i < nl * N; i += blockDim.x) {
      const int l = i / N, x = i - l * N;
      const Tin* r0 = u + (2 * (y0 + l)) * N + x;
      S0[i] = mk<T>((T)__ldg(r0), (T)__ldg(r0 + N));
    }
    __syncthreads();
    const cplx_t<T>* res = stockham<T>(S0, S1, nl, fr, tw);
    for (int i = threadIdx.x; i < nl * H; i += blockDim.x) {
      const int l = i / H, k = i - l * H;
      const cplx_t<T> Z = res[l * N + k], Zc = res[l * N + (N - k) % N];
      const int y = 2 * (y0 + l);
      P[y * H + k] = mk<T>(T(0.5) * (Z.x + Zc.x), T(0.5) * (Z.y - Zc.y));          // (Z + conj Zc) / 2
      P[(y + 1) * H + k] = mk<T>(T(0.5) * (Z.y + Zc.y), -T(0.5) * (Z.x - Zc.x));   // (Z - conj Zc) / (2i)
    }
    __syncthreads();
  }
  for (int k0 = 0; k0 < H; k0 += cwl) {
    const int nl = min(cwl, H - k0);
    for (int i = threadIdx.x; i < nl * N; i += blockDim.x) {
      const int l = i % nl, y = i / nl;
      S0[l * N + y] = P[y * H + k0 + l];
    }
    __syncthreads();
    const cplx_t<T>* res = stockham<T>(S0, S1, nl, fr, tw);
    for (int i = threadIdx.x; i < nl * N; i += blockDim.x) {
      const int l = i % nl, ky = i / nl;
      P[ky * H + k0 + l] = res[l * N + ky];
    }
    __syncthreads();
  }
  cplx_t<T>* o = out + (p * N + z) * (int64_t)N * H;
  for (int i = threadIdx.x; i < N * H; i += blockDim.x) o[i] = P[i];
}

// ---- stage 5b: correlation along z of the plane spectra, on the window only --------------------------------------
// With f~, rho~ the 2-D (x, y) spectra of the planes, the kz part of IFFT(F^ conj(rho^)) at integer tz is a circular
// correlation along z (no z transform needed):
//   Y1[p][a][ky][kx] = sum_z f~(kx, ky, (z + tz_a) mod N) conj(rho~(kx, ky, z)),   tz_a = a - (W + 1), a < w' = 2W+3
// One CTA per (ky row, kx chunk of hc, particle): both rows of every z are staged transposed ([kx][z], padded) and
// each output (kx, a) is an N-term complex dot product; outputs are staged and written as contiguous rows.
template <typename T>
__global__ void __launch_bounds__(256) k_zcorr(const cplx_t<T>* __restrict__ ft, const cplx_t<T>* __restrict__ rt,
                                               int N, int W, int hc, cplx_t<T>* __restrict__ Y1) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int H = N / 2 + 1, wp = 2 * W + 3, nkc = (H + hc - 1) / hc, ld = N + 1;
  cplx_t<T>* fs = reinterpret_cast<cplx_t<T>*>(smem_raw);  // [hc][N+1]
  cplx_t<T>* rs = fs + hc * ld;                             // [hc][N+1]
  const int ky = blockIdx.x / nkc, kx0 = (blockIdx.x - ky * nkc) * hc, nk = min(hc, H - kx0);
  const int64_t p = blockIdx.y;
  for (int i = threadIdx.x; i < N * nk; i += blockDim.x) {
    const int zz = i / nk, kl = i - zz * nk;
    const int64_t g = ((p * N + zz) * N + ky) * (int64_t)H + kx0 + kl;
    fs[kl * ld + zz] = ft[g];
    rs[kl * ld + zz] = rt[g];
  }
  __syncthreads();
  cplx_t<T> acc[4];  // nk * wp <= 4 * blockDim.x (zcorr_chunk)
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int o = threadIdx.x + u * blockDim.x;
    if (o >= nk * wp) break;
    const int kl = o / wp, a = o - kl * wp;
    const cplx_t<T>* fr = fs + kl * ld;
    const cplx_t<T>* rr = rs + kl * ld;
    int zz = ((a - (W + 1)) % N + N) % N;
    T ar = T(0), ai = T(0);
    for (int zi = 0; zi < N; ++zi) {
      const cplx_t<T> f = fr[zz], r = rr[zi];
      ar = fma(f.x, r.x, fma(f.y, r.y, ar));   // f conj(r)
      ai = fma(f.y, r.x, fma(-f.x, r.y, ai));
      if (++zz == N) zz = 0;
    }
    acc[u] = mk<T>(ar, ai);
  }
  __syncthreads();
  // stage [a][kl] in fs, then contiguous row writes Y1[p][a][ky][kx0 .. kx0 + nk)
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int o = threadIdx.x + u * blockDim.x;
    if (o >= nk * wp) break;
    const int kl = o / wp, a = o - kl * wp;
    fs[a * hc + kl] = acc[u];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < wp * nk; i += blockDim.x) {
    const int a = i / nk, kl = i - a * nk;
    Y1[((p * wp + a) * N + ky) * (int64_t)H + kx0 + kl] = fs[a * hc + kl];
  }
}

// ---- stage 5c: the (x, y) part of the window inverse, one CTA per (tz plane, particle) ----------------------------
//   cw[p][a][b][c] = Re sum_{ky} e^{+2 pi i ky ty_b / N} sum_{kx <= N/2} w_kx Y1[p][a][ky][kx] e^{+2 pi i kx tx_c / N}
// (w_kx = 1 at kx = 0 and N/2, else 2: the Hermitian half spectrum) = N^2 c(t) for t = (tx_c, ty_b, tz_a).
template <typename T>
__global__ void __launch_bounds__(512) k_window_xy(const cplx_t<T>* __restrict__ Y1, int N, int W, T* __restrict__ cw) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int H = N / 2 + 1, wp = 2 * W + 3;
  cplx_t<T>* base = reinterpret_cast<cplx_t<T>*>(smem_raw);  // [N] e^{+2 pi i j / N}
  cplx_t<T>* tw = base + N;                                  // [N][wp] e^{+2 pi i k t_a / N}
  cplx_t<T>* Y = tw + N * wp;                                // [N][H]
  cplx_t<T>* Z = Y + N * H;                                  // [N][wp]
  const int a = blockIdx.x;
  const int64_t p = blockIdx.y;
  build_roots<T>(base, N, +1);
  const cplx_t<T>* y1 = Y1 + (p * wp + a) * (int64_t)N * H;
  for (int i = threadIdx.x; i < N * H; i += blockDim.x) {
    const int kx = i % H;
    const T wk = (kx == 0 || 2 * kx == N) ? T(1) : T(2);
    const cplx_t<T> v = y1[i];
    Y[i] = mk<T>(wk * v.x, wk * v.y);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < N * wp; i += blockDim.x) {
    const int k = i / wp, t = i - k * wp - (W + 1);
    tw[i] = base[(((k * t) % N) + N) % N];
  }
  __syncthreads();
  for (int o = threadIdx.x; o < N * wp; o += blockDim.x) {
    const int ky = o / wp, c = o - ky * wp;
    const cplx_t<T>* yr = Y + ky * H;
    T ar = T(0), ai = T(0);
    for (int kx = 0; kx < H; ++kx) {
      const cplx_t<T> v = yr[kx], t = tw[kx * wp + c];
      ar = fma(v.x, t.x, fma(-v.y, t.y, ar));
      ai = fma(v.x, t.y, fma(v.y, t.x, ai));
    }
    Z[o] = mk<T>(ar, ai);
  }
  __syncthreads();
  for (int o = threadIdx.x; o < wp * wp; o += blockDim.x) {
    const int b = o / wp, c = o - b * wp;
    T ar = T(0);
    for (int ky = 0; ky < N; ++ky) {
      const cplx_t<T> v = Z[ky * wp + c], t = tw[ky * wp + b];
      ar = fma(v.x, t.x, fma(-v.y, t.y, ar));
    }
    cw[(p * wp + a) * (int64_t)wp * wp + o] = ar;
  }
}

// ---- stage 5d: windowed argmax (ties -> lowest window index, z-major) + per-axis parabolic subpixel (C18) -------
template <typename T>
__global__ void __launch_bounds__(256) k_window_peak(const T* __restrict__ cw_all, int N, int W, T* shifts,
                                                     int sstride, T* peak, int* __restrict__ tint) {
  __shared__ T sv[8];
  __shared__ int si[8];
  const int64_t p = blockIdx.x;
  const int wp = 2 * W + 3, w = 2 * W + 1;
  const T* cw = cw_all + p * (int64_t)wp * wp * wp;
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
      if (tint) tint[p * 3 + ax] = t[ax];
    }
    if (peak) peak[p] = c0 / ((T)N * N);
  }
}

// ==== FP32 fast path for the common box edges (N = 32, 64, 96, 128): compile-time FFT stages, the rotation fused
// into the transform of rho (texture gathers), register-blocked z correlation ====================================
__host__ __device__ constexpr int ct_nst(int n) {
  int s = 0;
  while (n % 8 == 0) { n /= 8; ++s; }
  while (n % 4 == 0) { n /= 4; ++s; }
  while (n % 2 == 0) { n /= 2; ++s; }
  while (n % 3 == 0) { n /= 3; ++s; }
  for (int r = 5; n > 1; r += 2)
    while (n % r == 0) { n /= r; ++s; }
  return s;
}
// k-th radix (same order as fft_radix) and the product of the radices before it
__host__ __device__ constexpr int ct_rad(int n, int k) {
  int s = 0;
  while (n % 8 == 0) { if (s++ == k) return 8; n /= 8; }
  while (n % 4 == 0) { if (s++ == k) return 4; n /= 4; }
  while (n % 2 == 0) { if (s++ == k) return 2; n /= 2; }
  while (n % 3 == 0) { if (s++ == k) return 3; n /= 3; }
  for (int r = 5; n > 1; r += 2)
    while (n % r == 0) { if (s++ == k) return r; n /= r; }
  return 1;
}
__host__ __device__ constexpr int ct_ns(int n, int k) {
  int p = 1;
  for (int i = 0; i < k; ++i) p *= ct_rad(n, i);
  return p;
}

constexpr int kFftThreads = 512;
// shared-memory index padding of the FFT line buffers: one float2 of slack every 16 (the radix-R stage writes at
// stride R and the transposes at stride N + 1; without it a warp's 8-byte stores hit 4 banks 4-way)
__host__ __device__ constexpr int fpad(int i) { return i + (i >> 4); }

// one Stockham stage on NL lines of length N at line stride LS (compile time: the index divisions are shifts/mults)
template <int N, int NL, int LS, int S>
__device__ __forceinline__ void ct_stage(const float2* __restrict__ a, float2* __restrict__ b,
                                         const float2* __restrict__ tw) {
  constexpr int R = ct_rad(N, S), Ns = ct_ns(N, S), NB = N / R, TS = N / (Ns * R), TOT = NL * NB;
#pragma unroll
  for (int t0 = 0; t0 < TOT; t0 += kFftThreads) {
    const int t = t0 + (int)threadIdx.x;
    if (TOT % kFftThreads != 0 && t >= TOT) break;
    const int l = t / NB, j = t - l * NB, k = j % Ns;
    const int ib = l * LS + j, ob = l * LS + (j - k) * R + k;
    if constexpr (R == 8) {
      // radix 8 in registers (one smem pass instead of two radix-4/2 passes): a = v_r + v_{r+4}, b = v_r - v_{r+4},
      // X[2q] = DFT4(a)[q], X[2q+1] = DFT4(b_r W8^r)[q], W8 = e^{-i pi/4}
      float2 v[8];
      v[0] = a[fpad(ib)];
#pragma unroll
      for (int r = 1; r < 8; ++r) v[r] = cmul<float>(a[fpad(ib + r * NB)], tw[r * k * TS]);
      const float h = 0.70710678118654752440f;
      float2 A4[4], B4[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        A4[r] = cadd<float>(v[r], v[r + 4]);
        B4[r] = csub<float>(v[r], v[r + 4]);
      }
      B4[1] = make_float2((B4[1].x + B4[1].y) * h, (B4[1].y - B4[1].x) * h);
      B4[2] = cmi<float>(B4[2]);
      B4[3] = make_float2((B4[3].y - B4[3].x) * h, (-B4[3].x - B4[3].y) * h);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const float2* u = half ? B4 : A4;
        const float2 s02 = cadd<float>(u[0], u[2]), d02 = csub<float>(u[0], u[2]), s13 = cadd<float>(u[1], u[3]),
                     d13 = cmi<float>(csub<float>(u[1], u[3]));
        b[fpad(ob + (0 + half) * Ns)] = cadd<float>(s02, s13);
        b[fpad(ob + (2 + half) * Ns)] = cadd<float>(d02, d13);
        b[fpad(ob + (4 + half) * Ns)] = csub<float>(s02, s13);
        b[fpad(ob + (6 + half) * Ns)] = csub<float>(d02, d13);
      }
    } else if constexpr (R == 4) {
      const float2 v0 = a[fpad(ib)], v1 = cmul<float>(a[fpad(ib + NB)], tw[k * TS]),
                   v2 = cmul<float>(a[fpad(ib + 2 * NB)], tw[2 * k * TS]),
                   v3 = cmul<float>(a[fpad(ib + 3 * NB)], tw[3 * k * TS]);
      const float2 s02 = cadd<float>(v0, v2), d02 = csub<float>(v0, v2), s13 = cadd<float>(v1, v3),
                   d13 = cmi<float>(csub<float>(v1, v3));
      b[fpad(ob)] = cadd<float>(s02, s13);
      b[fpad(ob + Ns)] = cadd<float>(d02, d13);
      b[fpad(ob + 2 * Ns)] = csub<float>(s02, s13);
      b[fpad(ob + 3 * Ns)] = csub<float>(d02, d13);
    } else if constexpr (R == 2) {
      const float2 v0 = a[fpad(ib)], v1 = cmul<float>(a[fpad(ib + NB)], tw[k * TS]);
      b[fpad(ob)] = cadd<float>(v0, v1);
      b[fpad(ob + Ns)] = csub<float>(v0, v1);
    } else {
      static_assert(R == 3, "fast path: radices 8, 4, 2, 3");
      const float2 v0 = a[fpad(ib)], v1 = cmul<float>(a[fpad(ib + NB)], tw[k * TS]),
                   v2 = cmul<float>(a[fpad(ib + 2 * NB)], tw[2 * k * TS]);
      const float h = 0.86602540378443864676f;
      const float2 sm = cadd<float>(v1, v2), df = csub<float>(v1, v2);
      const float2 m = make_float2(v0.x - 0.5f * sm.x, v0.y - 0.5f * sm.y);
      b[fpad(ob)] = cadd<float>(v0, sm);
      b[fpad(ob + Ns)] = make_float2(m.x + h * df.y, m.y - h * df.x);
      b[fpad(ob + 2 * Ns)] = make_float2(m.x - h * df.y, m.y + h * df.x);
    }
  }
}
template <int N, int NL, int LS, int S = 0>
__device__ __forceinline__ float2* ct_fft(float2* a, float2* b, const float2* tw) {
  if constexpr (S == ct_nst(N)) {
    return a;
  } else {
    ct_stage<N, NL, LS, S>(a, b, tw);
    __syncthreads();
    return ct_fft<N, NL, LS, S + 1>(b, a, tw);
  }
}

// buffer sizes (float2) with the fpad slack: the x pass runs in two halves of N/4 row pairs (A <-> B); the y pass
// ping-pongs C with A + B
template <int N> constexpr int plane_c() { return fpad((N / 2 + 1) * (N + 1)); }
template <int N> constexpr int plane_ab() {
  return fpad((N / 4) * N) > (plane_c<N>() + 1) / 2 ? fpad((N / 4) * N) : (plane_c<N>() + 1) / 2;
}
template <int N> constexpr size_t plane_fast_smem() {
  static_assert(2 * plane_ab<N>() >= plane_c<N>(), "the y pass ping-pongs C with A + B");
  return sizeof(float2) * ((size_t)N + 2 * (size_t)plane_ab<N>() + (size_t)plane_c<N>());
}

// 2-D R2C of every z-plane, FP32, compile-time N.  ROT = false: u = the particle volume (float [N][N][N]);
// ROT = true: u = rho_p(x) = h(R_p^T (x - c) + c) computed here from the reference through a 2-D texture over the
// zero-padded plane stack (row z (N+1) + y; row z (N+1) + N is zero; border = 0), two tld4 gathers per voxel (the
// 2 x 2 footprints of planes z0 and z0 + 1), with k_rotate_ref's exact trilinear arithmetic; rho never touches HBM.
template <int N, bool ROT>
__global__ void __launch_bounds__(kFftThreads, 2) k_plane_fft(const float* __restrict__ vol,
                                                              const cudaTextureObject_t* __restrict__ texs,
                                                              const int* __restrict__ tsel,
                                                              const float* __restrict__ euler, int estride,
                                                              float2* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int H = N / 2 + 1, LP = N + 1, NQ = N / 4;  // NQ row pairs per x half
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  float2* A = tw + N;              // [N/4][N] x-pass lines, then (with B) the y-pass ping-pong buffer (fpad indices)
  float2* B = A + plane_ab<N>();
  float2* C = B + plane_ab<N>();   // [H][LP]: y-pass lines (column kx of the half rows)
  __shared__ double Rm[9];
  const int z = blockIdx.x;
  const int64_t p = blockIdx.y;
  build_roots<float>(tw, N, -1);
  float r0 = 0.f, r1 = 0.f, r2 = 0.f, r3 = 0.f, r4 = 0.f, r5 = 0.f, r6 = 0.f, r7 = 0.f, r8 = 0.f;
  const float c = 0.5f * (float)(N - 1), uz = (float)z - c;
  cudaTextureObject_t tex = 0;
  if (ROT) {
    tex = texs[tsel ? tsel[p] : 0];  // the particle's template or the single reference
    if (threadIdx.x == 0) rot_matrix<float>(euler + p * estride, Rm);
    __syncthreads();
    r0 = (float)Rm[0], r1 = (float)Rm[1], r2 = (float)Rm[2], r3 = (float)Rm[3], r4 = (float)Rm[4],
    r5 = (float)Rm[5], r6 = (float)Rm[6], r7 = (float)Rm[7], r8 = (float)Rm[8];
  }
  const float* u = vol + (p * N + z) * (int64_t)N * N;
  for (int half = 0; half < 2; ++half) {
    const int lb = half * NQ;  // first row pair of this half
    if (ROT) {
      for (int i = threadIdx.x; i < NQ * N; i += kFftThreads) {
        const int l = i / N, x = i - l * N;
        float v2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float ux = (float)x - c, uy = (float)(2 * (lb + l) + h) - c;
          const float qx = fmaf(r0, ux, fmaf(r3, uy, r6 * uz)) + c;  // R^T v
          const float qy = fmaf(r1, ux, fmaf(r4, uy, r7 * uz)) + c;
          const float qz = fmaf(r2, ux, fmaf(r5, uy, r8 * uz)) + c;
          const float fx0 = floorf(qx), fy0 = floorf(qy), fz0 = floorf(qz);
          const int x0 = (int)fx0, y0 = (int)fy0, z0 = (int)fz0;
          const float fx = qx - fx0, fy = qy - fy0, fz = qz - fz0;
          const float tu = (float)x0 + 1.0f;
          float4 g0 = make_float4(0.f, 0.f, 0.f, 0.f), g1 = g0;
          // rows y0, y0 + 1 stay inside plane z0's N + 1 rows (the zero row / the border) only for -1 <= y0 <= N - 1;
          // beyond that both rows are outside the box
          const bool yin = (unsigned)(y0 + 1) <= (unsigned)N;
          if (yin && (unsigned)z0 < (unsigned)N)
            g0 = tex2Dgather<float4>(tex, tu, (float)(z0 * (N + 1) + y0) + 1.0f, 0);
          if (yin && (unsigned)(z0 + 1) < (unsigned)N)
            g1 = tex2Dgather<float4>(tex, tu, (float)((z0 + 1) * (N + 1) + y0) + 1.0f, 0);
          // gather order (scripts/tld4_probe.cu): x = (x0, y0+1), y = (x0+1, y0+1), z = (x0+1, y0), w = (x0, y0)
          const float c00 = fmaf(fx, g0.z - g0.w, g0.w);
          const float c01 = fmaf(fx, g0.y - g0.x, g0.x);
          const float c10 = fmaf(fx, g1.z - g1.w, g1.w);
          const float c11 = fmaf(fx, g1.y - g1.x, g1.x);
          const float c0 = fmaf(fy, c01 - c00, c00);
          const float c1 = fmaf(fy, c11 - c10, c10);
          v2[h] = fmaf(fz, c1 - c0, c0);
        }
        A[fpad(i)] = make_float2(v2[0], v2[1]);
      }
    } else {
      // all of the half plane's loads in flight before the first shared-memory store
      constexpr int IT = (NQ * N + kFftThreads - 1) / kFftThreads;
      float e0[IT], e1[IT];
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const int i = (int)threadIdx.x + it * kFftThreads, l = i / N, x = i - l * N;
        if (i < NQ * N) {
          e0[it] = __ldg(u + 2 * (lb + l) * N + x);
          e1[it] = __ldg(u + (2 * (lb + l) + 1) * N + x);
        }
      }
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const int i = (int)threadIdx.x + it * kFftThreads;
        if (i < NQ * N) A[fpad(i)] = make_float2(e0[it], e1[it]);
      }
    }
    __syncthreads();
    const float2* res = ct_fft<N, NQ, N>(A, B, tw);
    for (int i = threadIdx.x; i < NQ * H; i += kFftThreads) {
      const int l = i / H, k = i - l * H;
      const float2 Z = res[fpad(l * N + k)], Zc = res[fpad(l * N + (N - k) % N)];
      const int y = 2 * (lb + l);
      C[fpad(k * LP + y)] = make_float2(0.5f * (Z.x + Zc.x), 0.5f * (Z.y - Zc.y));
      C[fpad(k * LP + y + 1)] = make_float2(0.5f * (Z.y + Zc.y), -0.5f * (Z.x - Zc.x));
    }
    __syncthreads();
  }
  const float2* res2 = ct_fft<N, H, LP>(C, A, tw);
  float2* o = out + (p * N + z) * (int64_t)N * H;
  for (int i = threadIdx.x; i < N * H; i += kFftThreads) {
    const int ky = i / H, kx = i - ky * H;
    o[i] = res2[fpad(kx * LP + ky)];
  }
}

// zero-padded plane stack of the reference for the gathers: pad[(z (N+1) + y) * pitch + x] (row z (N+1) + N = 0)
__global__ void k_pad_ref(const float* __restrict__ ref, int N, int pitch, float* __restrict__ pad) {
  const int64_t n = (int64_t)N * (N + 1) * pitch;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % pitch);
    const int64_t row = i / pitch;
    const int z = (int)(row / (N + 1)), y = (int)(row % (N + 1));
    pad[i] = (x < N && y < N) ? ref[((int64_t)z * N + y) * N + x] : 0.f;
  }
}

// register-blocked z correlation: thread (z segment s, tz block bk of TB, kx): TB accumulators, a rolling window of
// TB f~ values (one new shared-memory load and one rho~ load per z for TB complex MACs); the S segment partials are
// summed in a fixed order (deterministic).
template <int TB>
__global__ void __launch_bounds__(512) k_zcorr_rb(const float2* __restrict__ ft, const float2* __restrict__ rt, int N,
                                                  int W, int hc, int S, float2* __restrict__ Y1) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int H = N / 2 + 1, wp = 2 * W + 3, nkc = (H + hc - 1) / hc, nblk = (wp + TB - 1) / TB;
  float2* fs = reinterpret_cast<float2*>(smem_raw);  // [N][hc]  (natural layout: lanes own consecutive kx)
  float2* rs = fs + N * hc;                           // [N][hc]
  const int ky = blockIdx.x / nkc, kx0 = (blockIdx.x - ky * nkc) * hc, nk = min(hc, H - kx0);
  const int64_t p = blockIdx.y;
  {
    // asynchronous 8-byte copies of the N row segments (one in flight per element, no register round trip)
    const int64_t row0 = (p * N * N + ky) * (int64_t)H + kx0;  // z = 0
    for (int i = threadIdx.x; i < N * nk; i += blockDim.x) {
      const int zz = i / nk, kl = i - zz * nk;
      const int64_t g = row0 + (int64_t)zz * N * H + kl;
      const unsigned df = (unsigned)__cvta_generic_to_shared(fs + zz * hc + kl);
      const unsigned dr = (unsigned)__cvta_generic_to_shared(rs + zz * hc + kl);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(df), "l"(ft + g));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dr), "l"(rt + g));
    }
    asm volatile("cp.async.wait_all;\n" ::);
  }
  __syncthreads();
  const int kl = threadIdx.x % hc, rest = threadIdx.x / hc, bk = rest % nblk, s = rest / nblk;
  const bool live = s < S && kl < nk;
  const int zseg = N / S, z0 = s * zseg, a0 = bk * TB;
  float2 acc[TB];
#pragma unroll
  for (int u = 0; u < TB; ++u) acc[u] = make_float2(0.f, 0.f);
  if (live) {
    const float2* fr = fs + kl;
    const float2* rr = rs + kl;
    float2 fw[TB];
    int zi = ((z0 + a0 - (W + 1)) % N + N) % N;
#pragma unroll
    for (int u = 0; u < TB; ++u) {
      fw[u] = fr[zi * hc];
      if (++zi == N) zi = 0;
    }
    for (int zz = z0; zz < z0 + zseg; ++zz) {
      const float2 r = rr[zz * hc];
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        acc[u].x = fmaf(fw[u].x, r.x, fmaf(fw[u].y, r.y, acc[u].x));  // f conj(r)
        acc[u].y = fmaf(fw[u].y, r.x, fmaf(-fw[u].x, r.y, acc[u].y));
      }
#pragma unroll
      for (int u = 0; u + 1 < TB; ++u) fw[u] = fw[u + 1];
      fw[TB - 1] = fr[zi * hc];
      if (++zi == N) zi = 0;
    }
  }
  __syncthreads();
  float2* part = fs;  // [S][wp][hc] (S wp <= 2 N: fits fs + rs)
  if (live) {
#pragma unroll
    for (int u = 0; u < TB; ++u)
      if (a0 + u < wp) part[(s * wp + a0 + u) * hc + kl] = acc[u];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < wp * nk; i += blockDim.x) {
    const int a = i / nk, k = i - a * nk;
    float2 v = part[a * hc + k];
    for (int q = 1; q < S; ++q) v = cadd<float>(v, part[(q * wp + a) * hc + k]);
    Y1[((p * wp + a) * N + ky) * (int64_t)H + kx0 + k] = v;
  }
}


// ==== stage 5e: subpixel refinement by an upsampled DFT (Guizar-Sicairos; App. C remark iii) ===
// Around the integer window peak t0 the correlation's real trigonometric interpolant (reading C27)
//   c~(t) = (1/N^3) sum_{k in [0,N)^3} F^(k) conj(rho^(k)) D(kx,tx) D(ky,ty) D(kz,tz)   (see ups_phase)
// is evaluated on t = t0 + (u - h) / kappa, u in [0, U)^3, U = 2h + 1, h = ceil(1.5 kappa), by three matrix-multiply
// DFTs; the result is the grid argmax (ties -> lowest index, z-major).  D(k, t0 + s) = e^{2 pi i k t0 / N} D(k, s) for
// the integer t0 (at the Nyquist index too: cos(pi (t0 + s)) = (-1)^t0 cos(pi s)), so the per-particle part is one
// phase e^{2 pi i (kx tx0 + ky ty0 + kz tz0) / N} folded into X, and the three DFT matrices D(k, s_u) are constants:
//   k_zfft_cross  3-D spectra from the plane spectra: the z FFT of f~ and rho~ pencils (Stockham in shared memory),
//                 X' = F^ conj(rho^) e^{2 pi i k.t0 / N} written over rho~ (never needed again this alternation);
//   k_ups_left    mode products with the constant D [U][N] (register-tiled GEMMs, 64-column tiles), each written with
//                 the next contracted axis outermost so that every product is one GEMM per particle:
//                 Z1[ky][uz][kx] = sum_kz D[uz][kz] X'[kz][ky][kx]   ([U x N] x [N x N H])
//                 Z2[uy][uz][kx] = sum_ky D[uy][ky] Z1[ky][uz][kx]   ([U x N] x [N x U H]);
//   k_ups_xmax    c~ = Re sum_kx w D[kx][ux] Z2[uy][uz][kx] (half spectrum in kx: w = 1 at kx = 0 and N/2, else 2;
//                 Re at the end makes the half sum exact for the Hermitian X) per 64-row block, block argmax;
//   k_ups_final   per particle: argmax over the blocks, t = t0 + (u - h)/kappa, peak = c~ / N^3.
// Contracting z, y, x in that order costs U N^2 H + U^2 N H + U^3 H complex MACs (39 M at 96^3, kappa = 16).

// z FFT of the plane spectra of one (ky row, kx chunk) -> X over rt
template <typename T>
__global__ void __launch_bounds__(256) k_zfft_cross(const cplx_t<T>* __restrict__ ft, cplx_t<T>* __restrict__ rt,
                                                    const __grid_constant__ FftRadix fr, int hc,
                                                    const int* __restrict__ tint) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = fr.n, H = N / 2 + 1, nkc = (H + hc - 1) / hc;
  cplx_t<T>* tw = reinterpret_cast<cplx_t<T>*>(smem_raw);
  cplx_t<T>* f0 = tw + N;          // [hc][N] lines along z
  cplx_t<T>* f1 = f0 + hc * N;
  cplx_t<T>* r0 = f1 + hc * N;
  cplx_t<T>* r1 = r0 + hc * N;
  const int ky = blockIdx.x / nkc, kx0 = (blockIdx.x - ky * nkc) * hc, nk = min(hc, H - kx0);
  const int64_t p = blockIdx.y;
  build_roots<T>(tw, N, -1);
  for (int i = threadIdx.x; i < N * nk; i += blockDim.x) {
    const int zz = i / nk, kl = i - zz * nk;
    const int64_t g = ((p * N + zz) * N + ky) * (int64_t)H + kx0 + kl;
    f0[kl * N + zz] = ft[g];
    r0[kl * N + zz] = rt[g];
  }
  __syncthreads();
  const cplx_t<T>* Fz = stockham<T>(f0, f1, nk, fr, tw);
  const cplx_t<T>* Rz = stockham<T>(r0, r1, nk, fr, tw);
  const int tx0 = tint[p * 3], ty0 = tint[p * 3 + 1], tz0 = tint[p * 3 + 2];
  for (int i = threadIdx.x; i < N * nk; i += blockDim.x) {
    const int kz = i / nk, kl = i - kz * nk;
    const cplx_t<T> f = Fz[kl * N + kz], r = Rz[kl * N + kz];
    const cplx_t<T> x = mk<T>(f.x * r.x + f.y * r.y, f.y * r.x - f.x * r.y);
    // e^{+2 pi i m / N} = conj(tw[m]),  m = k . t0 mod N
    const int m = (int)((((int64_t)(kx0 + kl) * tx0 + (int64_t)ky * ty0 + (int64_t)kz * tz0) % N + N) % N);
    const cplx_t<T> e = tw[m];
    rt[((p * N + kz) * N + ky) * (int64_t)H + kx0 + kl] = mk<T>(x.x * e.x + x.y * e.y, x.y * e.x - x.x * e.y);
  }
}

// FP32, compile-time N: the same z FFTs with ct_fft, cp.async-staged lines, one CTA per (ky row, particle)
template <int N, int MODE>  // MODE 0: F^ from f~; 1: also store F^ into fz; 2: F^ read from fz
__global__ void __launch_bounds__(kFftThreads, 1) k_zfft_cross_fast(const float2* __restrict__ ft,
                                                                    float2* __restrict__ rt,
                                                                    const int* __restrict__ tint,
                                                                    float2* __restrict__ fz) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int H = N / 2 + 1, LB = fpad(H * N);
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  float2* f0 = tw + N;  // [H][N] lines along z (fpad indices)
  float2* r0 = f0 + LB;
  float2* t1 = r0 + LB;  // ping-pong buffer shared by the two transforms
  const int ky = blockIdx.x;
  const int64_t p = blockIdx.y;
  build_roots<float>(tw, N, -1);
  const int64_t row0 = (p * N * N + ky) * (int64_t)H;
  for (int i = threadIdx.x; i < N * H; i += kFftThreads) {
    const int zz = i / H, kx = i - zz * H;
    const int64_t g = row0 + (int64_t)zz * N * H + kx;
    const unsigned df = (unsigned)__cvta_generic_to_shared(f0 + fpad(kx * N + zz));
    const unsigned dr = (unsigned)__cvta_generic_to_shared(r0 + fpad(kx * N + zz));
    // MODE 2: the cached F^ (kz in place of z), already transformed
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(df), "l"((MODE == 2 ? fz : ft) + g));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dr), "l"(rt + g));
  }
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  float2* Fz = MODE == 2 ? f0 : ct_fft<N, H, N>(f0, t1, tw);  // result in f0 or t1
  float2* rin = r0;
  float2* rtmp = (Fz == f0) ? t1 : f0;        // the buffer not holding F^
  // r0 -> rtmp -> r0 ...: ct_fft alternates the two buffers it is given
  const float2* Rz = ct_fft<N, H, N>(rin, rtmp, tw);
  const int tx0 = tint[p * 3], ty0 = tint[p * 3 + 1], tz0 = tint[p * 3 + 2];
  const int myz = ((ky * ty0) % N + N) % N;
  for (int i = threadIdx.x; i < N * H; i += kFftThreads) {
    const int kz = i / H, kx = i - kz * H;
    const float2 f = Fz[fpad(kx * N + kz)], r = Rz[fpad(kx * N + kz)];
    if (MODE == 1) fz[row0 + (int64_t)kz * N * H + kx] = f;
    const float2 x = make_float2(f.x * r.x + f.y * r.y, f.y * r.x - f.x * r.y);
    // the per-particle phase of the upsampled DFT: e^{+2 pi i m / N} = conj(tw[m]),  m = k . t0 mod N
    const int m = ((kx * tx0 + kz * tz0) % N + N + myz) % N;
    const float2 e = tw[m];
    rt[row0 + (int64_t)kz * N * H + kx] = make_float2(x.x * e.x + x.y * e.y, x.y * e.x - x.x * e.y);
  }
}

// interpolation kernel D(k, t) of reading C27: e^{+2 pi i k' t / N} with k' the symmetric frequency of index k
// (k' = k - N for k > N/2), and the real cos(pi t) at the Nyquist index k = N/2 (split evenly between +-N/2)
template <typename T> __device__ __forceinline__ cplx_t<T> ups_phase(int k, int N, int t0, int u, int h, int kappa) {
  const T t = (T)t0 + (T)(u - h) / (T)kappa;
  if (2 * k == N) {
    if constexpr (sizeof(T) == 8) return mk<T>(cospi(t), T(0));
    else return mk<T>(cospif(t), T(0));
  }
  const int kp = k < N / 2 ? k : k - N;
  T sn, cs;
  if constexpr (sizeof(T) == 8) sincospi(2.0 * kp * t / N, &sn, &cs);
  else sincospif(2.0f * (float)kp * t / (float)N, &sn, &cs);
  return mk<T>(cs, sn);
}

__host__ __device__ inline int ups_pad4(int U) { return (U + 3) / 4 * 4; }

constexpr int kUpsMaxU = 65;       // kappa <= 21
constexpr int kUpsThreads = 224;   // 208 active: 13 x 16 (left) or 16 x 13 (xmax) thread tiles of 4 x 4
constexpr int kUpsCols = 64;       // columns per CTA tile

// the constant DFT matrices, k-major: Dt [N][UP] = D(k, s_u) (reading C27 with t0 = 0; zero for u >= U),
// Dx [H][UP] = w(kx) D(kx, s_ux)
template <typename T>
__global__ void k_ups_tables(int N, int kappa, cplx_t<T>* __restrict__ Dt, cplx_t<T>* __restrict__ Dx) {
  const int H = N / 2 + 1, h = (int)ceil(1.5 * kappa), U = 2 * h + 1, UP = ups_pad4(U);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N * UP + H * UP; i += gridDim.x * blockDim.x) {
    if (i < N * UP) {
      const int k = i / UP, u = i - k * UP;
      Dt[i] = u < U ? ups_phase<T>(k, N, 0, u, h, kappa) : mk<T>(T(0), T(0));
    } else {
      const int j = i - N * UP, kx = j / UP, u = j - kx * UP;
      const T w = (kx == 0 || 2 * kx == N) ? T(1) : T(2);
      const cplx_t<T> e = u < U ? ups_phase<T>(kx, N, 0, u, h, kappa) : mk<T>(T(0), T(0));
      Dx[j] = mk<T>(w * e.x, w * e.y);
    }
  }
}

template <typename T> __host__ __device__ inline size_t ups_left_smem(int N, int U) {
  return sizeof(cplx_t<T>) * (size_t)N * (ups_pad4(U) + kUpsCols);
}

// out[s][u][c] = sum_{k < K} D[u][k] in[s][k][c]  (c < C; slice s = blockIdx.y, 64-column tile blockIdx.x): Dt
// [K][UP] and the input tile [K][64] staged by cp.async (zero fill past C), 4 (u) x 4 (c) complex outputs per thread
// (8 shared loads per 16 MACs)
template <typename T>
__global__ void __launch_bounds__(kUpsThreads) k_ups_left(const cplx_t<T>* __restrict__ Dt, int U, int K,
                                                          const cplx_t<T>* __restrict__ in, int64_t in_ss, int C,
                                                          cplx_t<T>* __restrict__ out, int64_t out_ss, int hs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int CS = (int)sizeof(cplx_t<T>);
  const int UP = ups_pad4(U);
  cplx_t<T>* Ds = reinterpret_cast<cplx_t<T>*>(smem_raw);  // [K][UP]
  cplx_t<T>* Is = Ds + K * UP;                                // [K][64]
  const int64_t sl = blockIdx.y;
  const int c0 = blockIdx.x * kUpsCols;
  {
    const unsigned char* dsrc = reinterpret_cast<const unsigned char*>(Dt);
    for (int e = threadIdx.x; e < K * UP * CS / 16; e += blockDim.x) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(reinterpret_cast<unsigned char*>(Ds) + 16 * e);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(dsrc + 16 * e));
    }
    const cplx_t<T>* src = in + sl * in_ss + c0;
    for (int i = threadIdx.x; i < K * kUpsCols; i += blockDim.x) {
      const int k = i / kUpsCols, c = i - k * kUpsCols;
      const bool ok = c0 + c < C;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(Is + i);
      const cplx_t<T>* g = ok ? src + (int64_t)k * C + c : src;
      if constexpr (CS == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0));
      else
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 16 : 0));
    }
    asm volatile("cp.async.wait_all;\n" ::);
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t >= 13 * 16) return;
  const int tu = t >> 4, tc = t & 15;
  T ar[4][4], ai[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) ar[i][j] = ai[i][j] = T(0);
  const cplx_t<T>* dp = Ds + 4 * tu;
  const cplx_t<T>* ip = Is + tc;
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    cplx_t<T> a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = dp[k * UP + i];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = ip[k * kUpsCols + 16 * j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        ar[i][j] = fma(a[i].x, b[j].x, fma(-a[i].y, b[j].y, ar[i][j]));
        ai[i][j] = fma(a[i].x, b[j].y, fma(a[i].y, b[j].x, ai[i][j]));
      }
  }
  // output layout: [u][c], or (hs > 0) [c / hs][u][c % hs] -- the next contraction's axis outermost
  cplx_t<T>* dst = out + sl * out_ss;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = c0 + tc + 16 * j;
    if (c >= C) continue;
    const int64_t base = hs ? (int64_t)(c / hs) * U * hs + c % hs : c;
    const int64_t ustep = hs ? hs : C;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int u = 4 * tu + i;
      if (u < U) dst[base + u * ustep] = mk<T>(ar[i][j], ai[i][j]);
    }
  }
}

template <typename T> __host__ __device__ inline size_t ups_xmax_smem(int N, int U) {
  const int H = N / 2 + 1;
  return sizeof(cplx_t<T>) * ((size_t)H * ups_pad4(U) + (size_t)kUpsCols * H);
}

// c~[r][ux] = Re sum_kx Z2[r][kx] Dx[kx][ux] for a block of 64 rows r = (uz, uy) of one particle (blockIdx.y), then
// the block's argmax (z-major index r U + ux, ties -> lowest) -> bval / bidx [particle][block]
template <typename T>
__global__ void __launch_bounds__(kUpsThreads) k_ups_xmax(const cplx_t<T>* __restrict__ Z2, const cplx_t<T>* __restrict__ Dx,
                                                          int N, int U, T* __restrict__ bval, int* __restrict__ bidx) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ T sv[kUpsThreads / 32];
  __shared__ int si[kUpsThreads / 32];
  const int H = N / 2 + 1, UP = ups_pad4(U), nrow = U * U;
  cplx_t<T>* Ds = reinterpret_cast<cplx_t<T>*>(smem_raw);  // [H][UP]
  cplx_t<T>* Zs = Ds + H * UP;                               // [64][H]
  const int64_t p = blockIdx.y;
  const int r0 = blockIdx.x * kUpsCols;
  for (int i = threadIdx.x; i < H * UP; i += blockDim.x) Ds[i] = Dx[i];
  const cplx_t<T>* src = Z2 + p * (int64_t)nrow * H;
  for (int i = threadIdx.x; i < kUpsCols * H; i += blockDim.x) {
    const int r = i / H;
    Zs[i] = r0 + r < nrow ? src[(int64_t)r0 * H + i] : mk<T>(T(0), T(0));
  }
  __syncthreads();
  const int t = threadIdx.x;
  T bv = -INFINITY;
  int bi = 0x7fffffff;
  if (t < 16 * 13) {
    const int tr = t / 13, tcol = t - tr * 13;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    const cplx_t<T>* zp = Zs + 4 * tr * H;
    const cplx_t<T>* dp = Ds + 4 * tcol;
#pragma unroll 4
    for (int k = 0; k < H; ++k) {
      cplx_t<T> z[4], d[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) z[i] = zp[i * H + k];
#pragma unroll
      for (int j = 0; j < 4; ++j) d[j] = dp[k * UP + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(z[i].x, d[j].x, fma(-z[i].y, d[j].y, acc[i][j]));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + 4 * tr + i, ux = 4 * tcol + j;  // r = uy U + uz
        const int idx = ((r % U) * U + r / U) * U + ux;    // z-major grid index uz U^2 + uy U + ux
        if (r < nrow && ux < U && better(acc[i][j], idx, bv, bi)) {
          bv = acc[i][j];
          bi = idx;
        }
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
  if ((t & 31) == 0) {
    sv[t >> 5] = bv;
    si[t >> 5] = bi;
  }
  __syncthreads();
  if (t == 0) {
    for (int k = 1; k < kUpsThreads / 32; ++k)
      if (better(sv[k], si[k], bv, bi)) {
        bv = sv[k];
        bi = si[k];
      }
    bval[p * gridDim.x + blockIdx.x] = bv;
    bidx[p * gridDim.x + blockIdx.x] = bi;
  }
}

template <typename T>
__global__ void k_ups_final(const T* __restrict__ bval, const int* __restrict__ bidx, int nblk, int N, int kappa,
                            const int* __restrict__ tint, int64_t nb, T* shifts, int sstride, T* peak) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nb) return;
  const int h = (int)ceil(1.5 * kappa), U = 2 * h + 1;
  T bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int k = 0; k < nblk; ++k)
    if (better(bval[p * nblk + k], bidx[p * nblk + k], bv, bi)) {
      bv = bval[p * nblk + k];
      bi = bidx[p * nblk + k];
    }
  const int u[3] = {bi % U, (bi / U) % U, bi / (U * U)};
  for (int ax = 0; ax < 3; ++ax) shifts[p * sstride + ax] = (T)tint[p * 3 + ax] + (T)(u[ax] - h) / (T)kappa;
  if (peak) peak[p] = bv / ((T)N * N * N);
}

}  // namespace

template <typename T>
cudaError_t launch_rotate_ref(const float* ref, int N, const T* euler, int estride, const int* tsel, int64_t nb, T* rho,
                              cudaStream_t s) {
  if (nb == 0) return cudaSuccess;
  const int64_t n3 = (int64_t)N * N * N;
  (void)n3;
  if (N % kRotTile) return cudaErrorInvalidValue;
  const int nt = N / kRotTile;
  k_rotate_ref<T><<<dim3((unsigned)std::min(nt * nt * nt, kRotCtas), (unsigned)nb), 256, 0, s>>>(ref, N, euler,
                                                                                                  estride, tsel, rho);
  return cudaGetLastError();
}

FftRadix fft_radix(int n) {
  FftRadix f;
  f.n = n;
  f.nst = 0;
  int m = n;
  for (int r : {4, 2, 3}) {
    while (m % r == 0 && f.nst < 16) {
      f.rad[f.nst++] = r;
      m /= r;
    }
  }
  for (int r = 5; m > 1 && f.nst < 16; r += 2)
    while (m % r == 0 && f.nst < 16) {
      f.rad[f.nst++] = r;
      m /= r;
    }
  return f;
}

static int plane_lines(int N, size_t csz) {
  const int H = N / 2 + 1;
  for (int cwl : {16, 8, 4, 2})
    if (csz * ((size_t)N + (size_t)N * H + 2 * (size_t)cwl * N) <= 227 * 1024) return cwl;
  return 0;
}
static size_t plane_smem(int N, int cwl, size_t csz) {
  return csz * ((size_t)N + (size_t)N * (N / 2 + 1) + 2 * (size_t)cwl * N);
}
static int zcorr_chunk(int N, int W, size_t csz) {
  const int H = N / 2 + 1, wp = 2 * W + 3;
  int hc = std::min(H, 1024 / wp);
  while (hc > 1 && 2 * csz * (size_t)hc * (N + 1) > 160 * 1024) --hc;
  return hc;
}
static size_t window_xy_smem(int N, int W, size_t csz) {
  const int wp = 2 * W + 3;
  return csz * ((size_t)N + 2 * (size_t)N * wp + (size_t)N * (N / 2 + 1));
}

bool trans_supported(int N, int W, bool fp64) {
  const size_t csz = fp64 ? 16 : 8;
  return plane_lines(N, csz) > 0 && 2 * W + 3 <= N && window_xy_smem(N, W, csz) <= 227 * 1024 &&
         zcorr_chunk(N, W, csz) >= 1;
}

template <typename T, typename Tin>
cudaError_t launch_plane_r2c(const Tin* vol, int N, int64_t nb, cplx_t<T>* out, cudaStream_t s) {
  if (nb == 0) return cudaSuccess;
  const size_t csz = sizeof(cplx_t<T>);
  const int cwl = plane_lines(N, csz);
  if (!cwl) return cudaErrorInvalidValue;
  const size_t smem = plane_smem(N, cwl, csz);
  cudaError_t e = cudaFuncSetAttribute(k_plane_r2c<T, Tin>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_plane_r2c<T, Tin><<<dim3((unsigned)N, (unsigned)nb), 256, smem, s>>>(vol, fft_radix(N), cwl, out);
  return cudaGetLastError();
}

bool plane_fast_supported(int N) { return N == 32 || N == 64 || N == 96 || N == 128; }

template <int N>
static cudaError_t launch_plane_fast(const float* vol, const cudaTextureObject_t* tex, const int* tsel,
                                     const float* euler, int estride, int64_t nb, float2* out, bool rot,
                                     cudaStream_t s) {
  constexpr size_t smem = plane_fast_smem<N>();
  static_assert(smem <= 227 * 1024, "plane buffers exceed shared memory");
  auto kern = rot ? k_plane_fft<N, true> : k_plane_fft<N, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3((unsigned)N, (unsigned)nb), kFftThreads, smem, s>>>(vol, tex, tsel, euler, estride, out);
  return cudaGetLastError();
}

cudaError_t launch_plane_fft_f32(const float* vol, const cudaTextureObject_t* tex, const int* tsel,
                                 const float* euler, int estride, int N, int64_t nb, float2* out, bool rot,
                                 cudaStream_t s) {
  if (nb == 0) return cudaSuccess;
  switch (N) {
    case 32: return launch_plane_fast<32>(vol, tex, tsel, euler, estride, nb, out, rot, s);
    case 64: return launch_plane_fast<64>(vol, tex, tsel, euler, estride, nb, out, rot, s);
    case 96: return launch_plane_fast<96>(vol, tex, tsel, euler, estride, nb, out, rot, s);
    case 128: return launch_plane_fast<128>(vol, tex, tsel, euler, estride, nb, out, rot, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_pad_ref(const float* ref, int N, int pitch, float* pad, cudaStream_t s) {
  k_pad_ref<<<592, 256, 0, s>>>(ref, N, pitch, pad);
  return cudaGetLastError();
}

size_t window_scratch_reals(int N, int W) {
  const int64_t wp = 2 * W + 3, H = N / 2 + 1;
  return (size_t)(2 * wp * N * H + wp * wp * wp);
}

// Y1 [nb][wp][N][H] complex at the front of the scratch, the c windows [nb][wp^3] behind it
template <typename T>
cudaError_t launch_window_zcorr(const cplx_t<T>* ft, const cplx_t<T>* rt, int N, int W, int64_t nb, T* scratch,
                                T* shifts, int sstride, T* peak, int* tint, cudaStream_t s) {
  if (nb == 0) return cudaSuccess;
  const size_t csz = sizeof(cplx_t<T>);
  if (!trans_supported(N, W, sizeof(T) == 8)) return cudaErrorInvalidValue;
  const int H = N / 2 + 1, wp = 2 * W + 3;
  const int hc = zcorr_chunk(N, W, csz), nkc = (H + hc - 1) / hc;
  cplx_t<T>* Y1 = reinterpret_cast<cplx_t<T>*>(scratch);
  T* cw = scratch + 2 * nb * (int64_t)wp * N * H;
  const size_t zsm = 2 * csz * (size_t)hc * (N + 1);
  cudaError_t e;
  if constexpr (sizeof(T) == 4) {
    constexpr int TB = 5;
    const int nblk = (wp + TB - 1) / TB;
    int S = 1;
    for (int q : {4, 3, 2})
      if (N % q == 0 && q * nblk * hc <= 512 && q * wp <= 2 * N) {
        S = q;
        break;
      }
    const int thr = std::min(512, (S * nblk * hc + 31) / 32 * 32);
    if (S * nblk * hc > 512) return cudaErrorInvalidValue;
    e = cudaFuncSetAttribute(k_zcorr_rb<TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zsm);
    if (e != cudaSuccess) return e;
    k_zcorr_rb<TB><<<dim3((unsigned)(N * nkc), (unsigned)nb), thr, zsm, s>>>(ft, rt, N, W, hc, S, Y1);
  } else {
    e = cudaFuncSetAttribute(k_zcorr<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zsm);
    if (e != cudaSuccess) return e;
    k_zcorr<T><<<dim3((unsigned)(N * nkc), (unsigned)nb), 256, zsm, s>>>(ft, rt, N, W, hc, Y1);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const size_t xsm = window_xy_smem(N, W, csz);
  e = cudaFuncSetAttribute(k_window_xy<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsm);
  if (e != cudaSuccess) return e;
  k_window_xy<T><<<dim3((unsigned)wp, (unsigned)nb), 512, xsm, s>>>(Y1, N, W, cw);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_window_peak<T><<<(unsigned)nb, 256, 0, s>>>(cw, N, W, shifts, sstride, peak, tint);
  return cudaGetLastError();
}

int ups_points(int kappa) { return 2 * (int)std::ceil(1.5 * kappa) + 1; }

size_t ups_scratch_bytes(int N, int kappa, size_t csz) {
  // per particle: Z1 [U][N][H] and the block bests; the constant tables D, Dx ride along (at most once per chunk)
  const size_t U = (size_t)ups_points(kappa), H = (size_t)N / 2 + 1;
  const size_t nblk = (U * U + kUpsCols - 1) / kUpsCols;
  return csz * (U * N * H) + nblk * (csz / 2 + sizeof(int)) + csz * ((size_t)N + H) * ups_pad4((int)U) + 256;
}

static int zfft_chunk(int N, size_t csz) {
  const int H = N / 2 + 1;
  int hc = H;
  while (hc > 1 && csz * ((size_t)N + 4 * (size_t)hc * N) > 200 * 1024) --hc;
  return hc;
}

bool ups_supported(int N, int kappa, bool fp64) {
  const size_t csz = fp64 ? 16 : 8;
  const int U = ups_points(kappa);
  const size_t lsm = fp64 ? ups_left_smem<double>(N, U) : ups_left_smem<float>(N, U);
  const size_t xsm = fp64 ? ups_xmax_smem<double>(N, U) : ups_xmax_smem<float>(N, U);
  return kappa >= 1 && U <= kUpsMaxU && lsm <= 200 * 1024 && xsm <= 200 * 1024 &&
         csz * ((size_t)N + 4 * (size_t)N) <= 200 * 1024;
}

// scratch: the tables Dt, Dx, then Z1 [nb][N][U][H], then the block bests; Z2 [nb][U][U][H] over X (rt);
// tint [nb][3] from k_window_peak
template <typename T>
cudaError_t launch_upsampled(const cplx_t<T>* ft, cplx_t<T>* rt, int N, int kappa, int64_t nb, const int* tint,
                             void* scratch, T* shifts, int sstride, T* peak, cudaStream_t s, cplx_t<T>* fz,
                             int fz_mode) {
  if (nb == 0) return cudaSuccess;
  const size_t csz = sizeof(cplx_t<T>);
  if (!ups_supported(N, kappa, sizeof(T) == 8)) return cudaErrorInvalidValue;
  const int H = N / 2 + 1, U = ups_points(kappa);
  const int hc = zfft_chunk(N, csz), nkc = (H + hc - 1) / hc;
  const size_t zsm = csz * ((size_t)N + 4 * (size_t)hc * N);
  cudaError_t e = cudaSuccess;
  bool fast = false;
  if constexpr (sizeof(T) == 4) {
    auto go = [&](auto kern, int NN) {
      const size_t sm = sizeof(float2) * ((size_t)NN + 3 * (size_t)fpad((NN / 2 + 1) * NN));
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e == cudaSuccess)
        kern<<<dim3((unsigned)NN, (unsigned)nb), kFftThreads, sm, s>>>(ft, rt, tint, (float2*)fz);
      fast = true;
    };
    const int md = fz ? fz_mode : 0;
    auto go3 = [&](auto k0, auto k1, auto k2, int NN) { md == 2 ? go(k2, NN) : md == 1 ? go(k1, NN) : go(k0, NN); };
    if (N == 32) go3(k_zfft_cross_fast<32, 0>, k_zfft_cross_fast<32, 1>, k_zfft_cross_fast<32, 2>, 32);
    else if (N == 64) go3(k_zfft_cross_fast<64, 0>, k_zfft_cross_fast<64, 1>, k_zfft_cross_fast<64, 2>, 64);
    else if (N == 96) go3(k_zfft_cross_fast<96, 0>, k_zfft_cross_fast<96, 1>, k_zfft_cross_fast<96, 2>, 96);
    else if (N == 128) go3(k_zfft_cross_fast<128, 0>, k_zfft_cross_fast<128, 1>, k_zfft_cross_fast<128, 2>, 128);
  }
  if (!fast) {
    e = cudaFuncSetAttribute(k_zfft_cross<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zsm);
    if (e != cudaSuccess) return e;
    k_zfft_cross<T><<<dim3((unsigned)(N * nkc), (unsigned)nb), 256, zsm, s>>>(ft, rt, fft_radix(N), hc, tint);
  }
  if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return e;
  const int UP = ups_pad4(U);
  cplx_t<T>* D = reinterpret_cast<cplx_t<T>*>(scratch);  // Dt [N][UP]
  cplx_t<T>* Dx = D + (size_t)N * UP;
  cplx_t<T>* Z1 = Dx + (size_t)H * UP;
  const int nblk = (U * U + kUpsCols - 1) / kUpsCols;
  T* bval = reinterpret_cast<T*>(Z1 + nb * (int64_t)U * N * H);
  int* bidx = reinterpret_cast<int*>(bval + nb * nblk);
  cplx_t<T>* Z2 = rt;  // X' is consumed by the z contraction
  k_ups_tables<T><<<(unsigned)((N * UP + H * UP + 255) / 256), 256, 0, s>>>(N, kappa, D, Dx);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const size_t lsm = ups_left_smem<T>(N, U);
  e = cudaFuncSetAttribute(k_ups_left<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm);
  if (e != cudaSuccess) return e;
  // z contraction: per particle [U x N] x [N x N H] -> Z1 [ky][uz][kx]
  const int cz = N * H;
  k_ups_left<T><<<dim3((unsigned)((cz + kUpsCols - 1) / kUpsCols), (unsigned)nb), kUpsThreads, lsm, s>>>(
      D, U, N, rt, (int64_t)N * N * H, cz, Z1, (int64_t)U * N * H, H);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // y contraction: per particle [U x N] x [N x U H] -> Z2 [uy][uz][kx]
  const int cy = U * H;
  k_ups_left<T><<<dim3((unsigned)((cy + kUpsCols - 1) / kUpsCols), (unsigned)nb), kUpsThreads, lsm, s>>>(
      D, U, N, Z1, (int64_t)N * U * H, cy, Z2, (int64_t)U * U * H, 0);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const size_t xsm = ups_xmax_smem<T>(N, U);
  e = cudaFuncSetAttribute(k_ups_xmax<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsm);
  if (e != cudaSuccess) return e;
  k_ups_xmax<T><<<dim3((unsigned)nblk, (unsigned)nb), kUpsThreads, xsm, s>>>(Z2, Dx, N, U, bval, bidx);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_ups_final<T><<<(unsigned)((nb + 127) / 128), 128, 0, s>>>(bval, bidx, nblk, N, kappa, tint, nb, shifts, sstride,
                                                               peak);
  return cudaGetLastError();
}

template cudaError_t launch_rotate_ref<float>(const float*, int, const float*, int, const int*, int64_t, float*,
                                              cudaStream_t);
template cudaError_t launch_rotate_ref<double>(const float*, int, const double*, int, const int*, int64_t, double*,
                                               cudaStream_t);
template cudaError_t launch_upsampled<float>(const float2*, float2*, int, int, int64_t, const int*, void*, float*, int,
                                             float*, cudaStream_t, float2*, int);
template cudaError_t launch_upsampled<double>(const double2*, double2*, int, int, int64_t, const int*, void*, double*,
                                              int, double*, cudaStream_t, double2*, int);
template cudaError_t launch_plane_r2c<float, float>(const float*, int, int64_t, float2*, cudaStream_t);
template cudaError_t launch_plane_r2c<double, float>(const float*, int, int64_t, double2*, cudaStream_t);
template cudaError_t launch_plane_r2c<double, double>(const double*, int, int64_t, double2*, cudaStream_t);
template cudaError_t launch_window_zcorr<float>(const float2*, const float2*, int, int, int64_t, float*, float*, int,
                                                float*, int*, cudaStream_t);
template cudaError_t launch_window_zcorr<double>(const double2*, const double2*, int, int, int64_t, double*, double*,
                                                 int, double*, int*, cudaStream_t);

}  // namespace matcha
