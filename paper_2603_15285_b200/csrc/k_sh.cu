// k_sh.cu -- stage 1: shell spherical-harmonic analysis of particle (and reference) volumes.
//
// north_star stage (1); PAPER.md P:109-111 (ball-harmonic expansion, separable radial x angular),
// P:1216-1220; readings C2-C5 (shells r_i = i - 1/2, Gauss-Legendre x equispaced quadrature with
// L_q = q L, orthonormal SH with Condon-Shortley phase, trilinear interpolation, zero outside):
//   f_lm(r_i) = sum_j W_j Pbar_lm(x_j) G_ijm,   G_ijm = (2pi/n_phi) sum_k u(c + t + r_i w_jk) e^{-i m phi_k}.
//
// B200 mapping (two kernels per sub-batch; the ring coefficients G of a sub-batch stay in the 126 MB L2):
//  k_sh_rings    one CTA per (particle, z-slab of S planes).  Every ring (r_i, theta_j) lies in ONE plane
//                pair (z = c_z + t_z + r_i cos theta_j), so the CTA stages its S+1 planes in shared memory
//                with coalesced 16-byte loads (the particle crosses HBM once, plus a 1/S halo) and does the
//                trilinear gathers of its rings from shared memory (rows padded to N+1 floats).  Each thread
//                gathers the 4 samples k, k+n/2, n/2-k, n-k of a ring and writes the real-data folds
//                (parity of m x cos/sin) k-major, so the DFT becomes four small real GEMMs
//                [rings x (Kh+1)] x [(Kh+1) x m] done with 2x4 register tiles against a precomputed
//                cos/sin table (~n_phi/4 FMAs per (ring, m) for Re and for Im, 4x fewer than a direct DFT).
//  k_sh_legendre one CTA per (particle, 4 shells): Legendre contraction with the node-pair fold
//                Pbar_lm(-x) = (-1)^{l+m} Pbar_lm(x) (G+ = G_j + G_j', G- = G_j - G_j' staged in shared
//                memory); thread tiles of (one m, 4 consecutive l) x 4 shells read the m-major weight table
//                W_j Pbar_lm(x_j) as float4.
// Deterministic: fixed summation orders, ring lists built by an ordered block scan, no atomics.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "common.cuh"

namespace matcha {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

constexpr int kRingThreads = 512;
constexpr int kRingWarps = kRingThreads / 32;
constexpr int kG = 8;  // rings per warp group (register tile of the DFT)

struct RingLayout {
  size_t tw, node, dft, pl, list, wsum, wbuf, total;
};

// staged plane rows are padded to N + 8 floats (16-byte aligned rows; bank = (8y + x) mod 32 at N = 64, the
// lowest bank-conflict degree of the quarter-arc gathers among the 16-byte-aligned pitches)
__host__ __device__ inline int plane_pitch(int N) { return N + 8; }

// per-warp fold buffer: [4 comps][Kh+1][kG] + mid [2][kG]
__host__ __device__ inline int wbuf_elems(int Kh) { return 4 * (Kh + 1) * kG + 2 * kG; }

template <typename T>
__host__ __device__ inline RingLayout ring_layout(int N, int S, int nth, int nph, int R, int Kh, int MP,
                                                   bool dft_smem = true, int warps = kRingWarps, bool staged = true) {
  RingLayout s;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t r = o;
    o += (b + 15) & ~size_t(15);
    return r;
  };
  s.tw = take(sizeof(cplx_t<T>) * nph);
  s.node = take(sizeof(cplx_t<T>) * nth);
  s.dft = take(dft_smem ? sizeof(cplx_t<T>) * (size_t)(Kh + 1) * MP : 0);
  s.pl = take(staged ? sizeof(float) * (size_t)(S + 1) * N * plane_pitch(N) : 0);
  s.list = take(sizeof(int) * (size_t)R * nth);
  s.wsum = take(sizeof(int) * (warps + 2));
  s.wbuf = take(sizeof(T) * (size_t)warps * wbuf_elems(Kh));
  s.total = o;
  return s;
}

// trilinear interpolation from the staged planes; pz0 = plane of floor(z) relative to the slab
template <typename T, int NT>
__device__ __forceinline__ T tri_smem(const float* __restrict__ pl, int Nr, int S, T px, T py, int pz0, T fz) {
  const int N = NT ? NT : Nr;
  const int W = plane_pitch(N), P = N * W;
  const T fx0 = floor(px), fy0 = floor(py);
  const int x0 = (int)fx0, y0 = (int)fy0;
  const T fx = px - fx0, fy = py - fy0;
  T c[2][2][2];
  if ((unsigned)x0 < (unsigned)(N - 1) && (unsigned)y0 < (unsigned)(N - 1) && (unsigned)pz0 < (unsigned)S) {
    const float* b = pl + pz0 * P + y0 * W + x0;
    c[0][0][0] = b[0];
    c[0][0][1] = b[1];
    c[0][1][0] = b[W];
    c[0][1][1] = b[W + 1];
    c[1][0][0] = b[P];
    c[1][0][1] = b[P + 1];
    c[1][1][0] = b[P + W];
    c[1][1][1] = b[P + W + 1];
  } else {
#pragma unroll
    for (int dz = 0; dz < 2; ++dz)
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
          const int x = x0 + dx, y = y0 + dy, z = pz0 + dz;
          const bool in = x >= 0 && y >= 0 && x < N && y < N && z >= 0 && z <= S;
          c[dz][dy][dx] = in ? (T)pl[z * P + y * W + x] : T(0);
        }
  }
  const T c00 = fma(fx, c[0][0][1] - c[0][0][0], c[0][0][0]);
  const T c01 = fma(fx, c[0][1][1] - c[0][1][0], c[0][1][0]);
  const T c10 = fma(fx, c[1][0][1] - c[1][0][0], c[1][0][0]);
  const T c11 = fma(fx, c[1][1][1] - c[1][1][0], c[1][1][0]);
  const T c0 = fma(fy, c01 - c00, c00);
  const T c1 = fma(fy, c11 - c10, c10);
  return fma(fz, c1 - c0, c0);
}

// large boxes (e.g. the paper's N = 200) whose plane slab does not fit shared memory: trilinear
// interpolation straight from the volume in global memory (read-only path; a ring's samples lie in one plane pair,
// so its gathers share L1 lines); z0 absolute, zero outside the box (reading C5)
template <typename T>
__device__ __forceinline__ T tri_glob(const float* __restrict__ v, int N, T px, T py, int z0, T fz) {
  const T fx0 = floor(px), fy0 = floor(py);
  const int x0 = (int)fx0, y0 = (int)fy0;
  const T fx = px - fx0, fy = py - fy0;
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

// four trilinear samples in one plane pair with a single bounds test, so the 32 shared-memory loads are
// issued back to back (ILP) on the common in-box path
template <typename T, int NT>
__device__ __forceinline__ void tri4(const float* __restrict__ pl, int Nr, int S, const T* px, const T* py, int pz0,
                                     T fz, T* out) {
  const int N = NT ? NT : Nr;
  const int W = plane_pitch(N), P = N * W;
  int x0[4], y0[4];
  T fx[4], fy[4];
  bool ok = (unsigned)pz0 < (unsigned)S;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const T fx0 = floor(px[i]), fy0 = floor(py[i]);
    x0[i] = (int)fx0;
    y0[i] = (int)fy0;
    fx[i] = px[i] - fx0;
    fy[i] = py[i] - fy0;
    ok = ok && (unsigned)x0[i] < (unsigned)(N - 1) && (unsigned)y0[i] < (unsigned)(N - 1);
  }
  if (ok) {
    float c[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float* b = pl + pz0 * P + y0[i] * W + x0[i];
      c[i][0] = b[0];
      c[i][1] = b[1];
      c[i][2] = b[W];
      c[i][3] = b[W + 1];
      c[i][4] = b[P];
      c[i][5] = b[P + 1];
      c[i][6] = b[P + W];
      c[i][7] = b[P + W + 1];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const T c00 = fma(fx[i], (T)c[i][1] - (T)c[i][0], (T)c[i][0]);
      const T c01 = fma(fx[i], (T)c[i][3] - (T)c[i][2], (T)c[i][2]);
      const T c10 = fma(fx[i], (T)c[i][5] - (T)c[i][4], (T)c[i][4]);
      const T c11 = fma(fx[i], (T)c[i][7] - (T)c[i][6], (T)c[i][6]);
      const T c0 = fma(fy[i], c01 - c00, c00);
      const T c1 = fma(fy[i], c11 - c10, c10);
      out[i] = fma(fz, c1 - c0, c0);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = tri_smem<T, NT>(pl, N, S, px[i], py[i], pz0, fz);
  }
}

template <typename T> struct V4;
template <> struct V4<float> {
  using t = float4;
};
template <> struct V4<double> {
  using t = double4;
};

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  const int n = valid ? 16 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(n));
}

template <typename T> __device__ __forceinline__ T warp_allsum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Ring DFT outputs of one warp group: lanes own m (rounds of 32); an isolated leftover m (<= 2 of them)
// is reduced across lanes instead of idling 30 lanes.
template <typename T>
__device__ __forceinline__ void group_dft(const T* __restrict__ wb, int nr, int Kh, int L, bool mid,
                                          const cplx_t<T>* __restrict__ dft, int MP, T dscale,
                                          cplx_t<T>* const* __restrict__ gout, int lane) {
  const int K1 = Kh + 1;
  const T* midv = wb + 4 * K1 * kG;
  int full = (L + 1) / 32, rem = (L + 1) - 32 * full;
  if (rem > 2) {
    ++full;
    rem = 0;
  }
  for (int c = 0; c < full; ++c) {
    const int m = 32 * c + lane;
    const bool act = m <= L;
    const int mm = act ? m : L;
    const int par = mm & 1;
    const T* P = wb + (2 * par) * K1 * kG;
    const T* Q = wb + (2 * par + 1) * K1 * kG;
    T re[kG], im[kG];
#pragma unroll
    for (int r = 0; r < kG; ++r) re[r] = im[r] = T(0);
    // twiddles (cos, sin)(m phi_k): reseeded from the table every 8 k, advanced by one complex rotation in
    // between (keeps shared-memory wavefronts for the fold operands; <= 8 ulp drift)
    const cplx_t<T> w1 = dft[1 * MP + mm];
    for (int k0 = 0; k0 < K1; k0 += 8) {
      cplx_t<T> w = dft[k0 * MP + mm];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int k = k0 + kk;
        if (k >= K1) break;
        const typename V4<T>::t p0 = *reinterpret_cast<const typename V4<T>::t*>(P + k * kG);
        const typename V4<T>::t p1 = *reinterpret_cast<const typename V4<T>::t*>(P + k * kG + 4);
        const typename V4<T>::t q0 = *reinterpret_cast<const typename V4<T>::t*>(Q + k * kG);
        const typename V4<T>::t q1 = *reinterpret_cast<const typename V4<T>::t*>(Q + k * kG + 4);
        const T pv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
        const T qv[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
        for (int r = 0; r < kG; ++r) {
          re[r] = fma(pv[r], w.x, re[r]);
          im[r] = fma(-qv[r], w.y, im[r]);
        }
        const T wx = w.x * w1.x - w.y * w1.y, wy = w.y * w1.x + w.x * w1.y;
        w = mk<T>(wx, wy);
      }
    }
    if (act)
#pragma unroll
      for (int r = 0; r < kG; ++r) {
        if (r >= nr) break;
        T vr = re[r], vi = im[r];
        if (mid) {
          const T am = midv[par * kG + r];
          switch (m & 3) {  // e^{-i m pi/2}
            case 0: vr += am; break;
            case 1: vi -= am; break;
            case 2: vr -= am; break;
            default: vi += am; break;
          }
        }
        gout[r][m] = mk<T>(vr * dscale, vi * dscale);
      }
  }
  // leftover m (at most 2): lanes = (ring r = lane % kG, k-quarter = lane / kG); each lane sums a quarter of the
  // k range, then two butterfly steps combine the quarters (fixed order)
  for (int e = 0; e < rem; ++e) {
    const int m = 32 * full + e, par = m & 1;
    const int r = lane % kG, qk = lane / kG;
    const T* P = wb + (2 * par) * K1 * kG + r;
    const T* Q = wb + (2 * par + 1) * K1 * kG + r;
    T vr = T(0), vi = T(0);
    for (int k = qk; k < K1; k += 32 / kG) {
      const cplx_t<T> w = dft[k * MP + m];
      vr = fma(P[k * kG], w.x, vr);
      vi = fma(-Q[k * kG], w.y, vi);
    }
#pragma unroll
    for (int o = kG; o < 32; o <<= 1) {
      vr += __shfl_xor_sync(0xffffffffu, vr, o);
      vi += __shfl_xor_sync(0xffffffffu, vi, o);
    }
    if (lane < nr) {
      if (mid) {
        const T am = midv[par * kG + r];
        switch (m & 3) {
          case 0: vr += am; break;
          case 1: vi -= am; break;
          case 2: vr -= am; break;
          default: vi += am; break;
        }
      }
      gout[lane][m] = mk<T>(vr * dscale, vi * dscale);
    }
  }
}

template <typename T, int NT, bool DFT_SMEM>
__global__ void __launch_bounds__(kRingThreads, 1) k_sh_rings(const float* __restrict__ vols,
                                                              const T* __restrict__ shifts, int shift_stride,
                                                              ShTables<T> tab, int S, int nslab,
                                                              cplx_t<T>* __restrict__ G) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr bool dft_smem = DFT_SMEM;
  constexpr bool GD = NT < 0;  // no plane staging: gathers straight from global memory (large boxes)
  const int N = NT > 0 ? NT : tab.N;
  const int R = tab.R, L = tab.L, nth = tab.nth, nph = tab.nph, Kh = tab.Kh, MP = tab.MP;
  const int Mp = nph / 2, K1 = Kh + 1;
  const bool mid = (Mp % 2) == 0;
  const int THR = blockDim.x, NW = THR / 32;  // 512 threads, fewer when shared memory is short (large Kh)
  const RingLayout lay = ring_layout<T>(N, S, nth, nph, R, Kh, MP, dft_smem, NW, !GD);
  cplx_t<T>* tw = (cplx_t<T>*)(smem + lay.tw);
  cplx_t<T>* node = (cplx_t<T>*)(smem + lay.node);
  const cplx_t<T>* dft = dft_smem ? (const cplx_t<T>*)(smem + lay.dft) : tab.dft;
  float* pl = (float*)(smem + lay.pl);
  int* list = (int*)(smem + lay.list);  // packed (i << 16) | j
  int* wsum = (int*)(smem + lay.wsum);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* wb = (T*)(smem + lay.wbuf) + (size_t)warp * wbuf_elems(Kh);

  const int64_t p = blockIdx.x / nslab;
  const int slab = blockIdx.x % nslab, zs = slab * S;
  const float* vol = vols + p * (int64_t)N * N * N;
  const T cc = T(0.5) * (T)(N - 1);
  T cx = cc, cy = cc, cz = cc;
  if (shifts) {
    cx += shifts[p * shift_stride + 0];
    cy += shifts[p * shift_stride + 1];
    cz += shifts[p * shift_stride + 2];
  }
  // 1. stage planes zs..zs+S asynchronously (cp.async 16 B, zero fill beyond the volume); each thread owns
  //    one 16-byte column x4 and walks rows with a fixed stride (no per-element division)
  if (!GD) {
    const int PW = plane_pitch(N), n4 = N / 4, rows = (S + 1) * N;
    if (THR % n4 == 0) {
      const int x4 = tid % n4, rstride = THR / n4;
      int row = tid / n4, pz = row / N, y = row - pz * N;
      for (; row < rows; row += rstride) {
        const int z = zs + pz;
        const bool valid = z < N;
        cp_async16(pl + (size_t)row * PW + 4 * x4, vol + ((size_t)(valid ? z : 0) * N + y) * N + 4 * x4, valid);
        y += rstride;
        while (y >= N) {
          y -= N;
          ++pz;
        }
      }
    } else {
      for (int t = tid; t < rows * n4; t += THR) {
        const int row = t / n4, x4 = t - row * n4, pz = row / N, y = row - pz * N, z = zs + pz;
        const bool valid = z < N;
        cp_async16(pl + (size_t)row * PW + 4 * x4, vol + ((size_t)(valid ? z : 0) * N + y) * N + 4 * x4, valid);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int t = tid; t < nph; t += THR) tw[t] = tab.tw[t];
  for (int t = tid; t < nth; t += THR) node[t] = tab.node[t];
  if (dft_smem)
    for (int t = tid; t < K1 * MP; t += THR) ((cplx_t<T>*)(smem + lay.dft))[t] = tab.dft[t];
  // 2. ordered list of the rings whose floor(z) belongs to this slab: one thread per node j counts its
  //    shells (z = c_z + r_i x_j is monotone in i), then an ordered scan over j (deterministic)
  int count = 0;
  {
    const int lo = (slab == 0) ? INT_MIN : zs, hi = (slab == nslab - 1) ? INT_MAX : zs + S;
    for (int j0 = 0; j0 < nth; j0 += THR) {
      const int j = j0 + tid;
      int cnt = 0;
      T xj = T(0);
      if (j < nth) {
        xj = tab.node[j].x;
        for (int i = 0; i < R; ++i) {
          const int zb = (int)floor(fma((T)i + T(0.5), xj, cz));
          cnt += (zb >= lo && zb < hi);
        }
      }
      int v = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (lane == 31) wsum[warp] = v;
      __syncthreads();
      int off = 0, tot = 0;
      for (int w = 0; w < NW; ++w) {
        if (w < warp) off += wsum[w];
        tot += wsum[w];
      }
      int pos = count + off + v - cnt;
      if (j < nth)
        for (int i = 0; i < R; ++i) {
          const int zb = (int)floor(fma((T)i + T(0.5), xj, cz));
          if (zb >= lo && zb < hi) list[pos++] = (i << 16) | j;
        }
      count += tot;
      __syncthreads();
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  // 3. warp-local work: a balanced contiguous range of rings per warp, in groups of kG
  const T dscale = T(2.0 * kPi) / (T)nph;
  const int r_begin = (int)(((long long)count * warp) / NW);
  const int r_end = (int)(((long long)count * (warp + 1)) / NW);
  for (int g0 = r_begin; g0 < r_end; g0 += kG) {
    const int nr = min(kG, r_end - g0);
    // folds: lanes walk consecutive k in [1, Kh] along ONE ring (gathers at neighbouring points: few bank
    // conflicts), 4 mirrored samples each; a lane keeps its 4 fold values of all kG rings in registers and writes
    // each k-row with two 16-byte stores.  k beyond the full rounds of 32 uses (ring, k) items spread over the
    // lanes; the k = 0 items (2 samples) are one sample per lane, combined by a shuffle.
    {
      auto ring_geom = [&](int r, T& rs, T& fz, int& pz0) {
        const int ring = list[g0 + r];
        const int i = ring >> 16, j = ring & 0xffff;
        const T rad = (T)i + T(0.5);
        const cplx_t<T> nd = node[j];
        rs = rad * nd.y;
        const T z = fma(rad, nd.x, cz);
        const T fz0 = floor(z);
        pz0 = (int)fz0 - zs;
        fz = z - fz0;
      };
      auto fold4 = [&](int k, T rs, T fz, int pz0, T* v) {
        const int kk[4] = {k, k + Mp, Mp - k, 2 * Mp - k};
        T px[4], py[4], sv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const cplx_t<T> ph = tw[kk[q]];
          px[q] = fma(rs, ph.x, cx);
          py[q] = fma(rs, ph.y, cy);
        }
        if constexpr (GD) {
#pragma unroll
          for (int q = 0; q < 4; ++q) sv[q] = tri_glob<T>(vol, N, px[q], py[q], pz0 + zs, fz);
        } else {
          tri4<T, NT>(pl, N, S, px, py, pz0, fz, sv);
        }
        const T ap = sv[0] + sv[1], am = sv[0] - sv[1], bp = sv[2] + sv[3], bm = sv[2] - sv[3];
        v[0] = ap + bp;  // even m, cos
        v[1] = ap - bp;  // even m, sin
        v[2] = am - bm;  // odd m, cos
        v[3] = am + bm;  // odd m, sin
      };
      const int nfull = Kh / 32;
      for (int kb = 0; kb < nfull * 32; kb += 32) {
        const int k = kb + lane + 1;
        T vals[4][kG];
#pragma unroll
        for (int r = 0; r < kG; ++r) {
          vals[0][r] = vals[1][r] = vals[2][r] = vals[3][r] = T(0);
          if (r < nr) {
            T rs, fz;
            int pz0;
            ring_geom(r, rs, fz, pz0);
            T v[4];
            fold4(k, rs, fz, pz0, v);
            vals[0][r] = v[0];
            vals[1][r] = v[1];
            vals[2][r] = v[2];
            vals[3][r] = v[3];
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          typename V4<T>::t* dst = reinterpret_cast<typename V4<T>::t*>(wb + (c * K1 + k) * kG);
          dst[0] = typename V4<T>::t{vals[c][0], vals[c][1], vals[c][2], vals[c][3]};
          dst[1] = typename V4<T>::t{vals[c][4], vals[c][5], vals[c][6], vals[c][7]};
        }
      }
      // leftover k in [32 nfull + 1, Kh]: items (ring r, k), r fastest
      const int kl0 = nfull * 32 + 1, nk = Kh - kl0 + 1;
      for (int it = lane; it < nk * kG; it += 32) {
        const int r = it % kG, k = kl0 + it / kG;
        T v[4] = {T(0), T(0), T(0), T(0)};
        if (r < nr) {
          T rs, fz;
          int pz0;
          ring_geom(r, rs, fz, pz0);
          fold4(k, rs, fz, pz0, v);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) wb[(c * K1 + k) * kG + r] = v[c];
      }
      // k = 0: samples phi = 0 and phi = pi (+ pi/2, 3pi/2 when the middle index exists), one per lane
      {
        const int r = lane >> 1, q = lane & 1;
        T s0 = T(0), sm = T(0);
        if (r < nr) {
          T rs, fz;
          int pz0;
          ring_geom(r, rs, fz, pz0);
          const cplx_t<T> ph = tw[q ? Mp : 0];
          if constexpr (GD) s0 = tri_glob<T>(vol, N, fma(rs, ph.x, cx), fma(rs, ph.y, cy), pz0 + zs, fz);
          else s0 = tri_smem<T, NT>(pl, N, S, fma(rs, ph.x, cx), fma(rs, ph.y, cy), pz0, fz);
          if (mid) {
            const cplx_t<T> pm = tw[Mp / 2 + (q ? Mp : 0)];
            if constexpr (GD) sm = tri_glob<T>(vol, N, fma(rs, pm.x, cx), fma(rs, pm.y, cy), pz0 + zs, fz);
            else sm = tri_smem<T, NT>(pl, N, S, fma(rs, pm.x, cx), fma(rs, pm.y, cy), pz0, fz);
          }
        }
        const T s1 = __shfl_xor_sync(0xffffffffu, s0, 1);
        const T sm1 = __shfl_xor_sync(0xffffffffu, sm, 1);
        if (q == 0 && r < kG) {
          wb[(0 * K1) * kG + r] = r < nr ? s0 + s1 : T(0);
          wb[(1 * K1) * kG + r] = T(0);
          wb[(2 * K1) * kG + r] = r < nr ? s0 - s1 : T(0);
          wb[(3 * K1) * kG + r] = T(0);
          if (mid) {
            wb[4 * K1 * kG + r] = sm + sm1;
            wb[4 * K1 * kG + kG + r] = sm - sm1;
          }
        }
      }
    }
    __syncwarp();
    cplx_t<T>* gout[kG];
#pragma unroll
    for (int r = 0; r < kG; ++r) {
      const int ring = list[g0 + min(r, nr - 1)];
      const int i = ring >> 16, j = ring & 0xffff;
      gout[r] = G + (((int64_t)p * R + i) * nth + j) * (L + 1);
    }
    group_dft<T>(wb, nr, Kh, L, mid, dft, MP, dscale, gout, lane);
    __syncwarp();
  }
}

struct LegLayout {
  size_t Gs, total;
};
template <typename T> __host__ __device__ inline LegLayout leg_layout(int SG, int JP, int L) {
  LegLayout s;
  size_t o = 0;
  s.Gs = o;
  o += sizeof(cplx_t<T>) * (size_t)2 * JP * SG * (L + 1);
  s.total = (o + 15) & ~size_t(15);
  return s;
}

// thread tiles of the parity-split layout: per m, ceil(#even / 4) + ceil(#odd / 4)
__host__ __device__ inline int leg_tiles_par(int L) {
  int n = 0;
  for (int m = 0; m <= L; ++m) n += ((L - m) / 2 + 1 + 3) / 4 + ((m + 1 <= L) ? ((L - m - 1) / 2 + 1 + 3) / 4 : 0);
  return n;
}

__host__ __device__ inline int leg_tiles(int L) {
  int n = 0;
  for (int m = 0; m <= L; ++m) n += (L - m + 4) / 4;
  return n;
}

// thread tile: one m, 4 consecutive l (l0t .. l0t+3), 4 shells; tiles enumerated m-major
template <typename T>
__global__ void __launch_bounds__(512) k_sh_legendre(const cplx_t<T>* __restrict__ G, ShTables<T> tab, int JP, cplx_t<T>* __restrict__ F) {
  constexpr int SG = 4;
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = tab.R, L = tab.L, nth = tab.nth, Jh = tab.Jh;
  const int ncf = ncoef(L);
  cplx_t<T>* Gs = (cplx_t<T>*)(smem);  // [2 (+,-)][JP][SG][L+1]
  const int ngroups = R / SG;
  const int64_t p = blockIdx.x / ngroups;
  const int i0 = (blockIdx.x % ngroups) * SG;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int ntiles = leg_tiles(L);
  const cplx_t<T>* Gp = G + (p * R) * (int64_t)nth * (L + 1);
  cplx_t<T>* Fp = F + p * (int64_t)ncf * R;
  for (int tile0 = 0; tile0 < ntiles; tile0 += nthr) {
    int m = -1, lb = 0;
    {
      int t = tile0 + tid;
      if (t < ntiles)
        for (int mm = 0; mm <= L; ++mm) {
          const int nt = (L - mm + 4) / 4;
          if (t < nt) {
            m = mm;
            lb = t;
            break;
          }
          t -= nt;
        }
    }
    const int l0t = (m >= 0) ? m + 4 * lb : 0;
    const int poff = (m >= 0) ? __ldg(&tab.pw_moff[m]) + 4 * lb : 0;
    T ar[4][SG], ai[4][SG];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int s = 0; s < SG; ++s) ar[a][s] = ai[a][s] = T(0);
    for (int q0 = 0; q0 < Jh; q0 += JP) {
      const int nq = min(JP, Jh - q0);
      __syncthreads();
      for (int t = tid; t < nq * SG * (L + 1); t += nthr) {
        const int mm = t % (L + 1), rest = t / (L + 1), s = rest % SG, q = rest / SG;
        const int jn = q0 + q, jm = nth - 1 - jn;
        const cplx_t<T> g1 = Gp[((int64_t)(i0 + s) * nth + jn) * (L + 1) + mm];
        cplx_t<T> g2 = mk<T>(T(0), T(0));
        if (jm != jn) g2 = Gp[((int64_t)(i0 + s) * nth + jm) * (L + 1) + mm];
        Gs[((0 * JP + q) * SG + s) * (L + 1) + mm] = mk<T>(g1.x + g2.x, g1.y + g2.y);
        Gs[((1 * JP + q) * SG + s) * (L + 1) + mm] = mk<T>(g1.x - g2.x, g1.y - g2.y);
      }
      __syncthreads();
      if (m < 0) continue;
      for (int q = 0; q < nq; ++q) {
        const typename V4<T>::t wv =
            *reinterpret_cast<const typename V4<T>::t*>(tab.pwm + (size_t)(q0 + q) * tab.pw_stride + poff);
        const T w[4] = {wv.x, wv.y, wv.z, wv.w};
        cplx_t<T> ge[SG], go[SG];  // parity of l+m: even uses G+, odd uses G-
#pragma unroll
        for (int s = 0; s < SG; ++s) {
          ge[s] = Gs[((0 * JP + q) * SG + s) * (L + 1) + m];
          go[s] = Gs[((1 * JP + q) * SG + s) * (L + 1) + m];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const bool odd = ((l0t + a + m) & 1) != 0;
#pragma unroll
          for (int s = 0; s < SG; ++s) {
            const cplx_t<T> g = odd ? go[s] : ge[s];
            ar[a][s] = fma(w[a], g.x, ar[a][s]);
            ai[a][s] = fma(w[a], g.y, ai[a][s]);
          }
        }
      }
    }
    if (m >= 0) {
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int l = l0t + a;
        if (l > L) continue;
        const int lm = l * (l + 1) / 2 + m;
#pragma unroll
        for (int s = 0; s < SG; ++s) Fp[(size_t)lm * R + i0 + s] = mk<T>(ar[a][s], ai[a][s]);
      }
    }
  }
}

// Legendre contraction, whole-shell-group variant: the CTA's SG shells of G (all nodes, all m) are copied to shared
// memory in one cp.async pass and node-pair folded in place (G_j +- G_{n-1-j}); thread tiles (one m, 4 consecutive l)
// x SG shells then stream the m-major weight rows W_j Pbar_lm(x_j) (float4, loaded two nodes ahead).
template <typename T> __host__ __device__ inline size_t leg_full_bytes(int SG, int nth, int L) {
  return sizeof(cplx_t<T>) * (size_t)SG * nth * (L + 1);
}

template <typename T, int SG, bool WS>
__global__ void __launch_bounds__(256) k_sh_legendre_full(const cplx_t<T>* __restrict__ G, ShTables<T> tab,
                                                          cplx_t<T>* __restrict__ F) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = tab.R, L = tab.L, nth = tab.nth, Jh = tab.Jh;
  const int L1 = L + 1, ncf = ncoef(L);
  cplx_t<T>* Gs = (cplx_t<T>*)smem;  // [SG][nth][L+1]
  const int ngroups = R / SG;
  const int64_t p = blockIdx.x / ngroups;
  const int i0 = (blockIdx.x % ngroups) * SG;
  const int tid = threadIdx.x, nthr = blockDim.x;
  {
    const cplx_t<T>* src = G + ((p * R + i0) * (int64_t)nth) * L1;
    const int nbytes = (int)sizeof(cplx_t<T>) * SG * nth * L1;
    const bool al16 = ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)nbytes) & 15) == 0;
    if (al16) {
      for (int e = tid; e < nbytes / 16; e += nthr) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared((unsigned char*)Gs + 16 * e);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"((const unsigned char*)src + 16 * e));
      }
    } else {
      for (int e = tid; e < nbytes / 8; e += nthr) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared((unsigned char*)Gs + 8 * e);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"((const unsigned char*)src + 8 * e));
      }
    }
    if (WS) {  // the whole m-major weight table W_j Pbar_lm(x_j), j < Jh (16-byte rows: pw_stride % 4 == 0)
      const int wbytes = (int)sizeof(T) * Jh * tab.pw_stride;
      unsigned char* wdst = smem + leg_full_bytes<T>(SG, nth, L);
      for (int e = tid; e < wbytes / 16; e += nthr) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(wdst + 16 * e);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"((const unsigned char*)tab.pwm + 16 * e));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  __syncthreads();
  {
    const int half = nth / 2;  // node pairs (j, nth-1-j), j < half; an odd middle node stays as is
    const uint32_t mgL = (uint32_t)((0x100000000ull + L1 - 1) / L1), mgH = (uint32_t)((0x100000000ull + half - 1) / half);
    for (int e = tid; e < SG * half * L1; e += nthr) {
      const int r = (int)__umulhi((uint32_t)e, mgL), m = e - r * L1;
      const int sh = (int)__umulhi((uint32_t)r, mgH), j = r - sh * half;
      cplx_t<T>* a = Gs + ((size_t)sh * nth + j) * L1 + m;
      cplx_t<T>* b = Gs + ((size_t)sh * nth + (nth - 1 - j)) * L1 + m;
      const cplx_t<T> u = *a, v = *b;
      *a = mk<T>(u.x + v.x, u.y + v.y);
      *b = mk<T>(u.x - v.x, u.y - v.y);
    }
  }
  __syncthreads();
  const int ntiles = leg_tiles(L);
  cplx_t<T>* Fp = F + p * (int64_t)ncf * R;
  using V = typename V4<T>::t;
  for (int tile = tid; tile < ntiles; tile += nthr) {
    int m = 0, lb = tile;
    for (; m <= L; ++m) {
      const int nt = (L - m + 4) / 4;
      if (lb < nt) break;
      lb -= nt;
    }
    const int l0t = m + 4 * lb;
    const int poff = __ldg(&tab.pw_moff[m]) + 4 * lb;
    const bool odd0 = ((l0t + m) & 1) != 0;  // parity of l + m for a = 0 (alternates with a)
    T ar[4][SG], ai[4][SG];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int s = 0; s < SG; ++s) ar[a][s] = ai[a][s] = T(0);
    const T* wrow = (WS ? (const T*)(smem + leg_full_bytes<T>(SG, nth, L)) : tab.pwm) + poff;
    constexpr int PD = 4;  // weight rows in flight
    V wq[PD];
#pragma unroll
    for (int u = 0; u < PD; ++u) wq[u] = *reinterpret_cast<const V*>(wrow + (size_t)min(u, Jh - 1) * tab.pw_stride);
    for (int q = 0; q < Jh; ++q) {
      const V wv = wq[0];
#pragma unroll
      for (int u = 0; u + 1 < PD; ++u) wq[u] = wq[u + 1];
      wq[PD - 1] = *reinterpret_cast<const V*>(wrow + (size_t)min(q + PD, Jh - 1) * tab.pw_stride);
      const T w[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
      for (int s = 0; s < SG; ++s) {
        const cplx_t<T> ge = Gs[((size_t)s * nth + q) * L1 + m];               // G+ (even l + m)
        const cplx_t<T> go = Gs[((size_t)s * nth + (nth - 1 - q)) * L1 + m];  // G- (odd l + m)
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const cplx_t<T> g = (odd0 ^ (a & 1)) ? go : ge;
          ar[a][s] = fma(w[a], g.x, ar[a][s]);
          ai[a][s] = fma(w[a], g.y, ai[a][s]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int l = l0t + a;
      if (l > L) continue;
      const int lm = l * (l + 1) / 2 + m;
#pragma unroll
      for (int s = 0; s < SG; ++s) Fp[(size_t)lm * R + i0 + s] = mk<T>(ar[a][s], ai[a][s]);
    }
  }
}

// Persistent Legendre (FP32): one CTA per SM holds the whole weight table W_j Pbar_lm(x_j) in shared memory (loaded
// once) and two independent 160-thread lanes, each walking its own (particle, 2-shell) items with the next item's G
// prefetched by cp.async into a second buffer while the current one is folded and contracted.
constexpr int kLegLaneThreads = 192;
constexpr int kLegSG = 2;

template <typename T>
__global__ void __launch_bounds__(2 * kLegLaneThreads, 1)
    k_sh_legendre_pers(const cplx_t<T>* __restrict__ G, ShTables<T> tab, int64_t nitems, cplx_t<T>* __restrict__ F) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int SG = kLegSG, LT = kLegLaneThreads;
  const int R = tab.R, L = tab.L, nth = tab.nth, Jh = tab.Jh;
  const int L1 = L + 1, ncf = ncoef(L);
  const int tid = threadIdx.x, lane_id = tid / LT, ltid = tid % LT;
  const size_t gbytes = sizeof(cplx_t<T>) * (size_t)SG * nth * L1;
  const int wbytes = (int)sizeof(T) * Jh * tab.pwp_stride;
  const T* W = (const T*)smem;
  // this lane's two G buffers (byte offsets into the dynamic shared memory: keeps every access an LDS/STS)
  const int gofs = (int)((((size_t)wbytes + 15) & ~size_t(15)) + (size_t)(2 * lane_id) * gbytes);
  auto gbuf = [&](int b) { return reinterpret_cast<cplx_t<T>*>(smem + gofs + b * (int)gbytes); };
  const int ngroups = R / SG;
  // this CTA's contiguous item range; lane l takes items l, l + 2, ...
  const int64_t i_begin = nitems * blockIdx.x / gridDim.x, i_end = nitems * (blockIdx.x + 1) / gridDim.x;
  // items are contiguous in G: one TMA bulk copy per item (issued by the lane's first thread, completion on a per-
  // (lane, buffer) mbarrier) when 16-byte aligned, else per-thread cp.async
  __shared__ __align__(8) uint64_t gmb[4];
  const bool bulk = ((gbytes & 15) == 0) && ((reinterpret_cast<uintptr_t>(G) & 15) == 0);
  if (tid == 0) {
    for (int b = 0; b < 4; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&gmb[b])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();
  auto copy_item = [&](int64_t it, int b) {
    cplx_t<T>* dst = gbuf(b);
    const int64_t p = it / ngroups;
    const int i0 = (int)(it % ngroups) * SG;
    const unsigned char* src = (const unsigned char*)(G + ((p * R + i0) * (int64_t)nth) * L1);
    if (bulk) {
      if (ltid == 0) {
        const unsigned bar = (unsigned)__cvta_generic_to_shared(&gmb[2 * lane_id + b]);
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("fence.proxy.async.shared::cta;\n" ::);  // the fold's writes to this buffer come first
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"((unsigned)gbytes)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         sa),
                     "l"(src), "r"((unsigned)gbytes), "r"(bar)
                     : "memory");
      }
      return;
    }
    const bool al16 = ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)gbytes) & 15) == 0;
    if (al16) {
      for (int e = ltid; e < (int)(gbytes / 16); e += LT) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared((unsigned char*)dst + 16 * e);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src + 16 * e));
      }
    } else {
      for (int e = ltid; e < (int)(gbytes / 8); e += LT) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared((unsigned char*)dst + 8 * e);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src + 8 * e));
      }
    }
  };
  for (int e = tid; e < wbytes / 16; e += 2 * LT) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem + 16 * e);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"((const unsigned char*)tab.pwp + 16 * e));
  }
  asm volatile("cp.async.commit_group;\n" ::);
  if (i_begin + lane_id < i_end) copy_item(i_begin + lane_id, 0);
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 1;\n" ::);  // this thread's part of the weight table
  const int ntiles = leg_tiles_par(L);
  __shared__ int tmap[kLegLaneThreads];            // thread tile -> (m, parity, l-block)
  __shared__ int toff[kLegLaneThreads];            // thread tile -> offset of its first weight in a W row
  for (int t = tid; t < ntiles; t += 2 * LT) {
    int m = 0, par = 0, lb = t;
    for (; m <= L; ++m) {
      const int ne = (L - m) / 2 + 1, no = (m + 1 <= L) ? (L - m - 1) / 2 + 1 : 0;
      const int te = (ne + 3) / 4, to = (no + 3) / 4;
      if (lb < te) { par = 0; break; }
      lb -= te;
      if (lb < to) { par = 1; break; }
      lb -= to;
    }
    tmap[t] = (lb << 17) | (par << 16) | m;
    toff[t] = tab.pwp_off[2 * m + par] + 4 * lb;
  }
  __syncthreads();                                // the whole weight table and the tile map
  const int half = nth / 2;
  const uint32_t mgL = (uint32_t)((0x100000000ull + L1 - 1) / L1), mgH = (uint32_t)((0x100000000ull + half - 1) / half);
  auto lbar = [&]() { asm volatile("bar.sync %0, %1;\n" ::"r"(1 + lane_id), "r"(LT)); };
  int k = 0;
  for (int64_t it = i_begin + lane_id; it < i_end; it += 2, ++k) {
    cplx_t<T>* Gs = gbuf(k & 1);
    if (it + 2 < i_end) copy_item(it + 2, (k + 1) & 1);
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 1;\n" ::);
    if (bulk) {  // the k/2-th fill of buffer k & 1 has landed
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&gmb[2 * lane_id + (k & 1)]);
      const unsigned ph = (unsigned)((k >> 1) & 1);
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}\n"
                     : "=r"(done)
                     : "r"(bar), "r"(ph)
                     : "memory");
    }
    lbar();
    // node-pair fold in place: (G_j, G_{n-1-j}) -> (G_j + G_{n-1-j}, G_j - G_{n-1-j})
    for (int e = ltid; e < SG * half * L1; e += LT) {
      const int r = (int)__umulhi((uint32_t)e, mgL), m = e - r * L1;
      const int sh = (int)__umulhi((uint32_t)r, mgH), j = r - sh * half;
      cplx_t<T>* a = Gs + (sh * nth + j) * L1 + m;
      cplx_t<T>* b = Gs + (sh * nth + (nth - 1 - j)) * L1 + m;
      const cplx_t<T> u = *a, v = *b;
      *a = mk<T>(u.x + v.x, u.y + v.y);
      *b = mk<T>(u.x - v.x, u.y - v.y);
    }
    lbar();
    const int64_t p = it / ngroups;
    const int i0 = (int)(it % ngroups) * SG;
    cplx_t<T>* Fp = F + p * (int64_t)ncf * R;
    {
      // this item's G is in shared memory now and nobody reads it again: drop its whole 128-byte L2 lines without
      // write-back (the two partial boundary lines are shared with the neighbouring items and stay)
      const uintptr_t g0 = reinterpret_cast<uintptr_t>(G + ((p * R + i0) * (int64_t)nth) * L1);
      const uintptr_t a0 = (g0 + 127) & ~uintptr_t(127), a1 = (g0 + gbytes) & ~uintptr_t(127);
      for (uintptr_t a = a0 + 128 * (uintptr_t)ltid; a < a1; a += 128 * (uintptr_t)LT)
        asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(a) : "memory");
    }
    for (int tile = ltid; tile < ntiles; tile += LT) {
      const int m = tmap[tile] & 0xffff, par = (tmap[tile] >> 16) & 1, lb = tmap[tile] >> 17;
      const int l0t = m + par + 8 * lb;  // degrees l0t, l0t + 2, l0t + 4, l0t + 6 (same parity of l - m)
      const T* wrow = W + toff[tile];
      T ar[4][SG], ai[4][SG];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int s2 = 0; s2 < SG; ++s2) ar[a][s2] = ai[a][s2] = T(0);
      using V = typename V4<T>::t;
      // G+ (even l - m) sits at node q, G- (odd) at node n-1-q after the fold
      const cplx_t<T>* g0 = Gs + (par ? (nth - 1) * L1 : 0) + m;
      const int gstep = par ? -L1 : L1, sstep = nth * L1;
#pragma unroll 3
      for (int q = 0; q < Jh; ++q) {
        const V wv = *reinterpret_cast<const V*>(wrow + (size_t)q * tab.pwp_stride);
        const T w[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int s2 = 0; s2 < SG; ++s2) {
          const cplx_t<T> g = g0[s2 * sstep + q * gstep];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            ar[a][s2] = fma(w[a], g.x, ar[a][s2]);
            ai[a][s2] = fma(w[a], g.y, ai[a][s2]);
          }
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int l = l0t + 2 * a;
        if (l > L) continue;
        const int lm = l * (l + 1) / 2 + m;
#pragma unroll
        for (int s2 = 0; s2 < SG; ++s2) Fp[(size_t)lm * R + i0 + s2] = mk<T>(ar[a][s2], ai[a][s2]);
      }
    }
    lbar();  // the buffer is refilled by the prefetch two items later
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
}

template <typename T> size_t leg_pers_bytes(const ShTables<T>& tab) {
  const size_t w = (sizeof(T) * (size_t)tab.Jh * tab.pwp_stride + 15) & ~size_t(15);
  return w + 4 * sizeof(cplx_t<T>) * (size_t)kLegSG * tab.nth * (tab.L + 1);
}

template <typename T> struct ShPlan {
  int S, nslab, threads;
  bool dft_smem;
  bool gd;  // no plane staging (box too large for a shared-memory slab)
  size_t rbytes;
};

template <typename T> ShPlan<T> sh_plan(const ShTables<T>& tab) {
  // one CTA per SM: the deepest slab (<= 8 planes) that fits with 16 warps; the DFT table moves to global memory
  // (read through L1) if shared memory cannot hold it; large boxes / degrees (e.g. 128^3, L = 64) use 8 or 4 warps
  ShPlan<T> pl;
  const size_t budget = 224 * 1024;
  for (int warps = kRingWarps; warps >= 2; warps /= 2)
    for (int pass = 0; pass < 2; ++pass) {
      const bool ds = (pass == 0);
      for (int S = 8; S >= 1; --S) {
        const size_t tot = ring_layout<T>(tab.N, S, tab.nth, tab.nph, tab.R, tab.Kh, tab.MP, ds, warps).total;
        if (tot <= budget) {
          pl.S = S;
          pl.dft_smem = ds;
          pl.gd = false;
          pl.nslab = (tab.N + S - 1) / S;
          pl.rbytes = tot;
          pl.threads = 32 * warps;
          return pl;
        }
      }
    }
  // no slab fits: gathers straight from global memory; slabs of 2 planes only group the rings, so that a CTA's
  // gathers stay within ~3 planes (L1 reuse: 200^3, L = 100: 19.8 vs 23.6 ms per 100 particles with 8-plane slabs)
  for (int warps = kRingWarps; warps >= 2; warps /= 2)
    for (int pass = 0; pass < 2; ++pass) {
      const bool ds = (pass == 0);
      const size_t tot = ring_layout<T>(tab.N, 2, tab.nth, tab.nph, tab.R, tab.Kh, tab.MP, ds, warps, false).total;
      if (tot <= budget) {
        pl.S = 2;
        pl.dft_smem = ds;
        pl.gd = true;
        pl.nslab = (tab.N + 1) / 2;
        pl.rbytes = tot;
        pl.threads = 32 * warps;
        return pl;
      }
    }
  pl.S = 2;
  pl.dft_smem = false;
  pl.gd = true;
  pl.nslab = (tab.N + 1) / 2;
  pl.threads = 64;
  pl.rbytes = ring_layout<T>(tab.N, 2, tab.nth, tab.nph, tab.R, tab.Kh, tab.MP, false, 2, false).total;
  return pl;
}

}  // namespace

template <typename T> size_t sh_ring_workspace_elems(const ShTables<T>& tab) {
  return (size_t)tab.R * tab.nth * (tab.L + 1);
}

template <typename T, int NT, bool DS>
static cudaError_t launch_rings_nt(const float* vols, int64_t nb, const T* shifts, int shift_stride,
                                   const ShTables<T>& tab, const ShPlan<T>& plan, cplx_t<T>* Gws, cudaStream_t st) {
  cudaError_t e =
      cudaFuncSetAttribute(k_sh_rings<T, NT, DS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.rbytes);
  if (e != cudaSuccess) return e;
  k_sh_rings<T, NT, DS><<<(unsigned)(nb * plan.nslab), plan.threads, plan.rbytes, st>>>(vols, shifts, shift_stride, tab,
                                                                                       plan.S, plan.nslab, Gws);
  return cudaGetLastError();
}

template <typename T, bool DS>
static cudaError_t launch_rings(const float* vols, int64_t nb, const T* shifts, int shift_stride,
                                const ShTables<T>& tab, const ShPlan<T>& plan, cplx_t<T>* Gws, cudaStream_t st) {
  if (plan.gd) return launch_rings_nt<T, -1, DS>(vols, nb, shifts, shift_stride, tab, plan, Gws, st);
  switch (tab.N) {  // compile-time box edges: immediate shared-memory offsets in the trilinear gathers
    case 16: return launch_rings_nt<T, 16, DS>(vols, nb, shifts, shift_stride, tab, plan, Gws, st);
    case 32: return launch_rings_nt<T, 32, DS>(vols, nb, shifts, shift_stride, tab, plan, Gws, st);
    case 64: return launch_rings_nt<T, 64, DS>(vols, nb, shifts, shift_stride, tab, plan, Gws, st);
    case 96: return launch_rings_nt<T, 96, DS>(vols, nb, shifts, shift_stride, tab, plan, Gws, st);
    case 128: return launch_rings_nt<T, 128, DS>(vols, nb, shifts, shift_stride, tab, plan, Gws, st);
    default: return launch_rings_nt<T, 0, DS>(vols, nb, shifts, shift_stride, tab, plan, Gws, st);
  }
}

template <typename T>
cudaError_t launch_sh_analysis(const float* vols, int64_t B, const T* shifts, int shift_stride, const ShTables<T>& tab,
                               cplx_t<T>* F, cplx_t<T>* Gws, int64_t gws_particles, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const int N = tab.N, ncf = ncoef(tab.L);
  const ShPlan<T> plan = sh_plan<T>(tab);
  const int JP = 8;
  const size_t lbytes = leg_layout<T>(4, JP, tab.L).total;
  const int lthreads = std::min(512, (leg_tiles(tab.L) + 31) / 32 * 32);
  cudaError_t e = cudaFuncSetAttribute(k_sh_legendre<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lbytes);
  if (e != cudaSuccess) return e;
  // whole-shell-group Legendre variant when SG shells of G fit in shared memory
  int lsg = 0;
  const size_t wtab = sizeof(T) * (size_t)tab.Jh * tab.pw_stride;
  if (tab.R % 8 == 0 && leg_full_bytes<T>(8, tab.nth, tab.L) + wtab <= 220 * 1024) lsg = 8;
  else if (tab.R % 4 == 0 && leg_full_bytes<T>(4, tab.nth, tab.L) <= 110 * 1024) lsg = 4;
  else if (tab.R % 2 == 0 && leg_full_bytes<T>(2, tab.nth, tab.L) <= 200 * 1024) lsg = 2;
  const bool lpers = sizeof(T) == 4 && tab.R % kLegSG == 0 && leg_tiles_par(tab.L) <= kLegLaneThreads &&
                     leg_pers_bytes<T>(tab) <= 226 * 1024;
  if (lpers) {
    e = cudaFuncSetAttribute(k_sh_legendre_pers<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)leg_pers_bytes<T>(tab));
    if (e != cudaSuccess) return e;
  }
  const size_t lfb = lsg ? leg_full_bytes<T>(lsg, tab.nth, tab.L) + (lsg == 8 ? wtab : 0) : 0;
  if (lsg == 8)
    e = cudaFuncSetAttribute(k_sh_legendre_full<T, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lfb);
  if (lsg == 4)
    e = cudaFuncSetAttribute(k_sh_legendre_full<T, 4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lfb);
  if (lsg == 2)
    e = cudaFuncSetAttribute(k_sh_legendre_full<T, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lfb);
  if (e != cudaSuccess) return e;
  const int lfthreads = std::min(256, (leg_tiles(tab.L) + 31) / 32 * 32);
  for (int64_t c0 = 0; c0 < B; c0 += gws_particles) {
    const int64_t nb = std::min<int64_t>(gws_particles, B - c0);
    const float* v = vols + c0 * (int64_t)N * N * N;
    const T* sh = shifts ? shifts + c0 * shift_stride : nullptr;
    if constexpr (sizeof(T) == 4) {
      // the persistent tensor-core kernel gives one particle to one SM: small batches (e.g. the reference) go to
      // the slab-parallel SIMT kernel instead, which spreads one particle over N/S CTAs
      if (tab.tcP > 0 && nb * 4 >= tab.num_sms)
        e = launch_sh_rings_tc(v, nb, sh, shift_stride, tab, tab.tcP, Gws, tab.flags, tab.num_sms, st);
      else {
        // small batches (e.g. the reference): thinner slabs, so that one particle still spreads over many SMs
        ShPlan<T> pl = plan;
        if (!pl.gd && nb * pl.nslab < tab.num_sms) {
          pl.S = std::max<int>(1, (int)((int64_t)pl.S * nb * pl.nslab / tab.num_sms));
          pl.nslab = (N + pl.S - 1) / pl.S;
        }
        e = pl.dft_smem ? launch_rings<T, true>(v, nb, sh, shift_stride, tab, pl, Gws, st)
                        : launch_rings<T, false>(v, nb, sh, shift_stride, tab, pl, Gws, st);
      }
    } else {
      e = plan.dft_smem ? launch_rings<T, true>(v, nb, sh, shift_stride, tab, plan, Gws, st)
                        : launch_rings<T, false>(v, nb, sh, shift_stride, tab, plan, Gws, st);
    }
    if (e != cudaSuccess) return e;
    if (lpers) {
      const int64_t items = nb * (tab.R / kLegSG);
      const int grid = (int)std::min<int64_t>(tab.num_sms, (items + 1) / 2);
      k_sh_legendre_pers<T><<<grid, 2 * kLegLaneThreads, leg_pers_bytes<T>(tab), st>>>(
          Gws, tab, items, F + c0 * (int64_t)ncf * tab.R);
    } else if (lsg == 8)
      k_sh_legendre_full<T, 8, true><<<(unsigned)(nb * (tab.R / 8)), lfthreads, lfb, st>>>(Gws, tab, F + c0 * (int64_t)ncf * tab.R);
    else if (lsg == 4)
      k_sh_legendre_full<T, 4, false><<<(unsigned)(nb * (tab.R / 4)), lfthreads, lfb, st>>>(Gws, tab, F + c0 * (int64_t)ncf * tab.R);
    else if (lsg == 2)
      k_sh_legendre_full<T, 2, false><<<(unsigned)(nb * (tab.R / 2)), lfthreads, lfb, st>>>(Gws, tab, F + c0 * (int64_t)ncf * tab.R);
    else
      k_sh_legendre<T><<<(unsigned)(nb * (tab.R / 4)), lthreads, lbytes, st>>>(Gws, tab, JP,
                                                                                F + c0 * (int64_t)ncf * tab.R);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template size_t sh_ring_workspace_elems<float>(const ShTables<float>&);
template size_t sh_ring_workspace_elems<double>(const ShTables<double>&);
template cudaError_t launch_sh_analysis<float>(const float*, int64_t, const float*, int, const ShTables<float>&,
                                               float2*, float2*, int64_t, cudaStream_t);
template cudaError_t launch_sh_analysis<double>(const float*, int64_t, const double*, int, const ShTables<double>&,
                                                double2*, double2*, int64_t, cudaStream_t);

}  // namespace matcha
