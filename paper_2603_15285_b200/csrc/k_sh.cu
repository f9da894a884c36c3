// k_sh.cu -- stage 1: shell spherical-harmonic analysis of particle (and reference) volumes.
//
// north_star stage (1); PAPER.md P:109-111 (ball-harmonic expansion, separable radial x angular),
// P:1216-1220; readings C2-C5 (shells r_i = i - 1/2, Gauss-Legendre x equispaced quadrature with
// L_q = q L, orthonormal SH with Condon-Shortley phase, trilinear interpolation, zero outside):
//   f_lm(r_i) = sum_j W_j Pbar_lm(x_j) (2pi/n_phi) sum_k u(c + t + r_i w_jk) e^{-i m phi_k}.
//
// B200 mapping.  One CTA per (particle, group of SG shells); the volume (1 MiB at 64^3) crosses HBM
// once per particle: the CTAs of one particle are adjacent in the grid so the trilinear gathers of its
// 8 shell groups hit L2/L1.  Rings are processed in chunks of JP Gauss-Legendre node PAIRS (x_j, -x_j):
//   (a) gather the 2 JP rings of a shell into shared memory (fast path without bounds checks);
//   (b) real-data folding of each ring: s_k +- s_{k+n/2} selects the parity of m, then the pairing
//       k <-> n/2 - k turns the length-n_phi complex DFT into ~n_phi/4 real FMAs per (ring, m) for Re and
//       for Im (4x fewer than a direct DFT);
//   (c) Legendre contraction with the node-pair fold Pbar_lm(-x) = (-1)^{l+m} Pbar_lm(x): one table row
//       W_j Pbar_lm(x_j) per PAIR, shared by the SG shells of the CTA (table traffic / SG).
// Deterministic: fixed summation order, no atomics.
#include "common.cuh"

namespace matcha {

namespace {

constexpr int kThreads = 256;

template <typename T> struct ShLayout {
  size_t tw, node, S, Qb, G, acc, total;
};

template <typename T> __host__ __device__ inline ShLayout<T> sh_layout(int nph, int nth, int JP, int SG, int L, int ncf) {
  ShLayout<T> s;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t r = o;
    o += (b + 15) & ~size_t(15);
    return r;
  };
  const int Mp = nph / 2, Kh = (Mp - 1) / 2;
  s.tw = take(sizeof(cplx_t<T>) * nph);
  s.node = take(sizeof(cplx_t<T>) * nth);
  s.S = take(sizeof(T) * 2 * JP * nph);
  s.Qb = take(sizeof(T) * 2 * JP * (4 * Kh + 4));
  s.G = take(sizeof(cplx_t<T>) * SG * 2 * JP * (L + 1));
  s.acc = take(sizeof(cplx_t<T>) * SG * ncf);
  s.total = o;
  return s;
}

template <typename T>
__device__ __forceinline__ T trilinear(const float* __restrict__ v, int N, T px, T py, T pz) {
  const T fx0 = floor(px), fy0 = floor(py), fz0 = floor(pz);
  const int x0 = (int)fx0, y0 = (int)fy0, z0 = (int)fz0;
  const T fx = px - fx0, fy = py - fy0, fz = pz - fz0;
  T c[2][2][2];
  if (x0 >= 0 && y0 >= 0 && z0 >= 0 && x0 + 1 < N && y0 + 1 < N && z0 + 1 < N) {
    const float* b = v + ((size_t)z0 * N + y0) * N + x0;
    const size_t NN = (size_t)N * N;
    c[0][0][0] = __ldg(b);
    c[0][0][1] = __ldg(b + 1);
    c[0][1][0] = __ldg(b + N);
    c[0][1][1] = __ldg(b + N + 1);
    c[1][0][0] = __ldg(b + NN);
    c[1][0][1] = __ldg(b + NN + 1);
    c[1][1][0] = __ldg(b + NN + N);
    c[1][1][1] = __ldg(b + NN + N + 1);
  } else {
#pragma unroll
    for (int dz = 0; dz < 2; ++dz)
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
          const int x = x0 + dx, y = y0 + dy, z = z0 + dz;
          const bool in = x >= 0 && y >= 0 && z >= 0 && x < N && y < N && z < N;
          c[dz][dy][dx] = in ? (T)__ldg(v + ((size_t)z * N + y) * N + x) : T(0);
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

template <typename T>
__global__ void __launch_bounds__(kThreads) k_sh_analysis(const float* __restrict__ vols, int64_t B,
                                                          const T* __restrict__ shifts, int shift_stride,
                                                          ShTables<T> tab, int JP, int SG,
                                                          cplx_t<T>* __restrict__ F) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int N = tab.N, R = tab.R, L = tab.L, nth = tab.nth, nph = tab.nph, Jh = tab.Jh;
  const int ncf = ncoef(L);
  const int Mp = nph / 2, Kh = (Mp - 1) / 2;
  const bool mid = (Mp % 2) == 0;  // self-paired phi index Mp/2 exists
  const ShLayout<T> lay = sh_layout<T>(nph, nth, JP, SG, L, ncf);
  cplx_t<T>* tw = (cplx_t<T>*)(smem + lay.tw);
  cplx_t<T>* node = (cplx_t<T>*)(smem + lay.node);
  T* S = (T*)(smem + lay.S);
  T* Qb = (T*)(smem + lay.Qb);
  cplx_t<T>* G = (cplx_t<T>*)(smem + lay.G);
  cplx_t<T>* acc = (cplx_t<T>*)(smem + lay.acc);
  const int QW = 4 * Kh + 4;  // folded ring record: a0+, a0-, E[Kh], F[Kh], Gc[Kh], Hs[Kh], mid+, mid-

  const int ngroups = R / SG;
  const int64_t p = blockIdx.x / ngroups;
  const int i0 = (blockIdx.x % ngroups) * SG;
  const float* vol = vols + p * (int64_t)N * N * N;
  const T cc = T(0.5) * (T)(N - 1);
  T cx = cc, cy = cc, cz = cc;
  if (shifts) {
    cx += shifts[p * shift_stride + 0];
    cy += shifts[p * shift_stride + 1];
    cz += shifts[p * shift_stride + 2];
  }
  for (int t = threadIdx.x; t < nph; t += kThreads) tw[t] = tab.tw[t];
  for (int t = threadIdx.x; t < nth; t += kThreads) node[t] = tab.node[t];
  for (int t = threadIdx.x; t < SG * ncf; t += kThreads) acc[t] = mk<T>(T(0), T(0));
  __syncthreads();

  const T dscale = T(2.0 * kPi) / (T)nph;
  for (int jp0 = 0; jp0 < Jh; jp0 += JP) {
    for (int s = 0; s < SG; ++s) {
      const T r = (T)(i0 + s) + T(0.5);
      // (a) gather rings (2q: node jn, 2q+1: mirrored node nth-1-jn)
      for (int t = threadIdx.x; t < 2 * JP * nph; t += kThreads) {
        const int rr = t / nph, k = t - rr * nph;
        const int jn = jp0 + (rr >> 1);
        const int j = (rr & 1) ? (nth - 1 - jn) : jn;
        T val = T(0);
        if (jn < Jh && !((rr & 1) && j == jn)) {
          const cplx_t<T> nd = node[j];  // (cos th, sin th)
          const cplx_t<T> ph = tw[k];    // (cos phi, sin phi)
          const T rs = r * nd.y;
          val = trilinear<T>(vol, N, fma(rs, ph.x, cx), fma(rs, ph.y, cy), fma(r, nd.x, cz));
        }
        S[rr * nph + k] = val;
      }
      __syncthreads();
      // (b1) parity / pair folding of each ring
      for (int t = threadIdx.x; t < 2 * JP * (Kh + 1); t += kThreads) {
        const int rr = t / (Kh + 1), k = t - rr * (Kh + 1);
        const T* sr = S + rr * nph;
        T* qb = Qb + rr * QW;
        if (k == 0) {
          qb[0] = sr[0] + sr[Mp];
          qb[1] = sr[0] - sr[Mp];
          if (mid) {
            const int km = Mp / 2;
            qb[2 + 4 * Kh] = sr[km] + sr[km + Mp];
            qb[3 + 4 * Kh] = sr[km] - sr[km + Mp];
          }
        } else {
          const int k2 = Mp - k;
          const T ap = sr[k] + sr[k + Mp], am = sr[k] - sr[k + Mp];
          const T bp = sr[k2] + sr[k2 + Mp], bm = sr[k2] - sr[k2 + Mp];
          qb[2 + (k - 1)] = ap + bp;           // even m, cos
          qb[2 + Kh + (k - 1)] = ap - bp;      // even m, sin
          qb[2 + 2 * Kh + (k - 1)] = am - bm;  // odd m, cos
          qb[2 + 3 * Kh + (k - 1)] = am + bm;  // odd m, sin
        }
      }
      __syncthreads();
      // (b2) G_m = a0 + sum_k [cos(m phi_k) P_k - i sin(m phi_k) Q_k] (+ self-paired term)
      for (int t = threadIdx.x; t < 2 * JP * (L + 1); t += kThreads) {
        const int rr = t / (L + 1), m = t - rr * (L + 1);
        const T* qb = Qb + rr * QW;
        const bool odd = m & 1;
        const T* Pc = qb + 2 + (odd ? 2 * Kh : 0);
        const T* Ps = qb + 2 + (odd ? 3 * Kh : Kh);
        T re = odd ? qb[1] : qb[0], im = T(0);
        int idx = 0;
        for (int k = 1; k <= Kh; ++k) {
          idx += m;
          if (idx >= nph) idx -= nph;
          const cplx_t<T> w = tw[idx];
          re = fma(w.x, Pc[k - 1], re);
          im = fma(-w.y, Ps[k - 1], im);
        }
        if (mid) {
          const T am = odd ? qb[3 + 4 * Kh] : qb[2 + 4 * Kh];
          switch (m & 3) {  // e^{-i m pi/2}
            case 0: re += am; break;
            case 1: im -= am; break;
            case 2: re -= am; break;
            default: im += am; break;
          }
        }
        G[(s * 2 * JP + rr) * (L + 1) + m] = mk<T>(re * dscale, im * dscale);
      }
      __syncthreads();
    }
    // (c) Legendre contraction for the SG shells, one table row per node pair
    for (int lm = threadIdx.x; lm < ncf; lm += kThreads) {
      int l = (int)((sqrtf(8.0f * lm + 1.0f) - 1.0f) * 0.5f);
      while (l * (l + 1) / 2 > lm) --l;
      while ((l + 1) * (l + 2) / 2 <= lm) ++l;
      const int m = lm - l * (l + 1) / 2;
      const T sg = ((l + m) & 1) ? T(-1) : T(1);
      cplx_t<T> a[8];
      for (int s = 0; s < SG; ++s) a[s] = acc[s * ncf + lm];
      for (int q = 0; q < JP && jp0 + q < Jh; ++q) {
        const T w = __ldg(&tab.pw[(size_t)(jp0 + q) * ncf + lm]);
        for (int s = 0; s < SG; ++s) {
          const cplx_t<T> g1 = G[(s * 2 * JP + 2 * q) * (L + 1) + m];
          const cplx_t<T> g2 = G[(s * 2 * JP + 2 * q + 1) * (L + 1) + m];
          a[s].x = fma(w, fma(sg, g2.x, g1.x), a[s].x);
          a[s].y = fma(w, fma(sg, g2.y, g1.y), a[s].y);
        }
      }
      for (int s = 0; s < SG; ++s) acc[s * ncf + lm] = a[s];
    }
    __syncthreads();
  }
  // write F[p][lm][i0 + s]
  cplx_t<T>* Fp = F + p * (int64_t)ncf * R;
  for (int t = threadIdx.x; t < SG * ncf; t += kThreads) {
    const int lm = t / SG, s = t - lm * SG;
    Fp[(size_t)lm * R + i0 + s] = acc[s * ncf + lm];
  }
}

}  // namespace

template <typename T>
cudaError_t launch_sh_analysis(const float* vols, int64_t B, const T* shifts, int shift_stride, const ShTables<T>& tab,
                               cplx_t<T>* F, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const int ncf = ncoef(tab.L);
  const int nchunks = (tab.Jh + 7) / 8;
  const int JP = (tab.Jh + nchunks - 1) / nchunks;
  int SG = 1;
  for (int cand : {4, 2, 1}) {
    if (tab.R % cand) continue;
    if (sh_layout<T>(tab.nph, tab.nth, JP, cand, tab.L, ncf).total <= 200 * 1024) {
      SG = cand;
      break;
    }
  }
  const size_t bytes = sh_layout<T>(tab.nph, tab.nth, JP, SG, tab.L, ncf).total;
  cudaError_t e = cudaFuncSetAttribute(k_sh_analysis<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  const int64_t blocks = B * (tab.R / SG);
  k_sh_analysis<T><<<(unsigned)blocks, kThreads, bytes, st>>>(vols, B, shifts, shift_stride, tab, JP, SG, F);
  return cudaGetLastError();
}

template cudaError_t launch_sh_analysis<float>(const float*, int64_t, const float*, int, const ShTables<float>&,
                                               float2*, cudaStream_t);
template cudaError_t launch_sh_analysis<double>(const float*, int64_t, const double*, int, const ShTables<double>&,
                                                double2*, cudaStream_t);

}  // namespace matcha
