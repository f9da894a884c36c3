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

#include "common.cuh"

namespace matcha {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

constexpr int kRingThreads = 512;
constexpr int kRingWarps = kRingThreads / 32;

struct RingLayout {
  size_t tw, node, dft, pl, list, wsum, fold, mid, total;
};

// staged plane rows are padded to N + 4 floats (16-byte aligned rows for cp.async; bank = (4y + x) mod 32)
__host__ __device__ inline int plane_pitch(int N) { return N + 4; }

template <typename T>
__host__ __device__ inline RingLayout ring_layout(int N, int S, int nth, int nph, int R, int RB, int Kh, int MP,
                                                   bool dft_smem = true) {
  RingLayout s;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t r = o;
    o += (b + 15) & ~size_t(15);
    return r;
  };
  s.tw = take(sizeof(cplx_t<T>) * nph);
  s.node = take(sizeof(cplx_t<T>) * nth);
  s.dft = take(dft_smem ? sizeof(T) * 4 * (size_t)(Kh + 1) * MP : 0);
  s.pl = take(sizeof(float) * (size_t)(S + 1) * N * plane_pitch(N));
  s.list = take(sizeof(int) * (size_t)R * nth);
  s.wsum = take(sizeof(int) * (kRingWarps + 2));
  s.fold = take(sizeof(T) * 4 * (size_t)(Kh + 1) * RB);
  s.mid = take(sizeof(T) * 2 * RB);
  s.total = o;
  return s;
}

// trilinear interpolation from the staged planes; pz0 = plane of floor(z) relative to the slab
template <typename T>
__device__ __forceinline__ T tri_smem(const float* __restrict__ pl, int N, int S, T px, T py, int pz0, T fz) {
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

template <typename T> struct V4;
template <> struct V4<float> {
  using t = float4;
};
template <> struct V4<double> {
  using t = double4;
};
template <typename T> struct V2;
template <> struct V2<float> {
  using t = float2;
};
template <> struct V2<double> {
  using t = double2;
};

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  const int n = valid ? 16 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(n));
}

template <typename T>
__global__ void __launch_bounds__(kRingThreads) k_sh_rings(const float* __restrict__ vols,
                                                           const T* __restrict__ shifts, int shift_stride,
                                                           ShTables<T> tab, int S, int nslab, int RB,
                                                           bool dft_smem, cplx_t<T>* __restrict__ G) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int N = tab.N, R = tab.R, L = tab.L, nth = tab.nth, nph = tab.nph, Kh = tab.Kh, MP = tab.MP;
  const int Mp = nph / 2;
  const bool mid = (Mp % 2) == 0;
  const RingLayout lay = ring_layout<T>(N, S, nth, nph, R, RB, Kh, MP, dft_smem);
  cplx_t<T>* tw = (cplx_t<T>*)(smem + lay.tw);
  cplx_t<T>* node = (cplx_t<T>*)(smem + lay.node);
  const T* dft = dft_smem ? (const T*)(smem + lay.dft) : tab.dft;  // [p][cs][k][MP]
  float* pl = (float*)(smem + lay.pl);
  int* list = (int*)(smem + lay.list);  // packed (i << 16) | j
  int* wsum = (int*)(smem + lay.wsum);
  T* fold = (T*)(smem + lay.fold);  // [4: Pe, Qe, Po, Qo][k][RB]
  T* midv = (T*)(smem + lay.mid);   // [2][RB]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

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
  {
    const int PW = plane_pitch(N), n4 = N / 4, rows = (S + 1) * N;
    if (kRingThreads % n4 == 0) {
      const int x4 = tid % n4, rstride = kRingThreads / n4;
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
      for (int t = tid; t < rows * n4; t += kRingThreads) {
        const int row = t / n4, x4 = t - row * n4, pz = row / N, y = row - pz * N, z = zs + pz;
        const bool valid = z < N;
        cp_async16(pl + (size_t)row * PW + 4 * x4, vol + ((size_t)(valid ? z : 0) * N + y) * N + 4 * x4, valid);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int t = tid; t < nph; t += kRingThreads) tw[t] = tab.tw[t];
  for (int t = tid; t < nth; t += kRingThreads) node[t] = tab.node[t];
  if (dft_smem)
    for (int t = tid; t < 4 * (Kh + 1) * MP; t += kRingThreads) ((T*)(smem + lay.dft))[t] = tab.dft[t];
  // 2. ordered list of the rings whose floor(z) belongs to this slab: one thread per node j counts its
  //    shells (z = c_z + r_i x_j is monotone in i), then an ordered scan over j (deterministic)
  int count = 0;
  {
    const int lo = (slab == 0) ? INT_MIN : zs, hi = (slab == nslab - 1) ? INT_MAX : zs + S;
    for (int j0 = 0; j0 < nth; j0 += kRingThreads) {
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
      // block exclusive scan of cnt
      int v = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (lane == 31) wsum[warp] = v;
      __syncthreads();
      int off = 0, tot = 0;
      for (int w = 0; w < kRingWarps; ++w) {
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
  const T dscale = T(2.0 * kPi) / (T)nph;
  const int nm0 = L / 2 + 1, nm1 = (L + 1) / 2;  // number of even / odd m in [0, L]
  const int mt0 = (nm0 + 3) / 4, mt1 = (nm1 + 3) / 4;
  // 3. batches of RB rings: gather + fold (one warp per ring, lanes over k), then the tiled real GEMMs
  for (int b0 = 0; b0 < count; b0 += RB) {
    const int nb = min(RB, count - b0);
    // items (ring rr, k in [0, Kh]) flattened over the CTA; (rr, k) advanced incrementally
    {
      const int K1 = Kh + 1;
      const int drr = kRingThreads / K1, dk = kRingThreads - drr * K1;
      int rr = tid / K1, k = tid - rr * K1;
      for (; rr < nb;) {
        const int ring = list[b0 + rr];
        const int i = ring >> 16, j = ring & 0xffff;
        const T r = (T)i + T(0.5);
        const cplx_t<T> nd = node[j];
        const T rs = r * nd.y;
        const T z = fma(r, nd.x, cz);
        const T fz0 = floor(z);
        const int pz0 = (int)fz0 - zs;
        const T fz = z - fz0;
        auto samp = [&](int kk) {
          const cplx_t<T> ph = tw[kk];
          return tri_smem<T>(pl, N, S, fma(rs, ph.x, cx), fma(rs, ph.y, cy), pz0, fz);
        };
        const bool k0 = (k == 0);
        const int k2 = Mp - k;
        const T s1 = samp(k), s2 = samp(k + Mp);
        const T s3 = k0 ? T(0) : samp(k2), s4 = k0 ? T(0) : samp(k2 + Mp);
        const T ap = s1 + s2, am = s1 - s2, bp = s3 + s4, bm = s3 - s4;
        fold[(0 * K1 + k) * RB + rr] = ap + bp;               // even m, cos
        fold[(1 * K1 + k) * RB + rr] = k0 ? T(0) : ap - bp;   // even m, sin
        fold[(2 * K1 + k) * RB + rr] = am - bm;               // odd m, cos
        fold[(3 * K1 + k) * RB + rr] = k0 ? T(0) : am + bm;   // odd m, sin
        if (k0 && mid) {
          const int km = Mp / 2;
          const T a = samp(km), bb = samp(km + Mp);
          midv[rr] = a + bb;
          midv[RB + rr] = a - bb;
        }
        rr += drr;
        k += dk;
        if (k >= K1) {
          k -= K1;
          ++rr;
        }
      }
    }
    __syncthreads();
    // tiles: (parity, m-tile of 4, ring-pair)
    const int rt = RB / 2;
    const int ntile = (mt0 + mt1) * rt;
    for (int t = tid; t < ntile; t += kRingThreads) {
      const int mtl = t / rt, rp = t - mtl * rt;
      const int par = mtl >= mt0 ? 1 : 0;
      const int mt = par ? mtl - mt0 : mtl;
      if (2 * rp >= nb) continue;
      const T* P = fold + (2 * par) * (Kh + 1) * RB + 2 * rp;
      const T* Q = fold + (2 * par + 1) * (Kh + 1) * RB + 2 * rp;
      const T* C = dft + ((par * 2 + 0) * (Kh + 1)) * MP + 4 * mt;
      const T* Sn = dft + ((par * 2 + 1) * (Kh + 1)) * MP + 4 * mt;
      T re[2][4], im[2][4];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) re[a][b] = im[a][b] = T(0);
#pragma unroll 4
      for (int k = 0; k <= Kh; ++k) {
        const typename V2<T>::t pv = *reinterpret_cast<const typename V2<T>::t*>(P + k * RB);
        const typename V2<T>::t qv = *reinterpret_cast<const typename V2<T>::t*>(Q + k * RB);
        const typename V4<T>::t cv = *reinterpret_cast<const typename V4<T>::t*>(C + k * MP);
        const typename V4<T>::t sv = *reinterpret_cast<const typename V4<T>::t*>(Sn + k * MP);
        const T pr[2] = {pv.x, pv.y}, qr[2] = {qv.x, qv.y};
        const T cr[4] = {cv.x, cv.y, cv.z, cv.w}, sr[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            re[a][b] = fma(pr[a], cr[b], re[a][b]);
            im[a][b] = fma(-qr[a], sr[b], im[a][b]);
          }
      }
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int rr = 2 * rp + a;
        if (rr >= nb) continue;
        const int ring = list[b0 + rr];
        const int i = ring >> 16, j = ring & 0xffff;
        cplx_t<T>* Gr = G + (((int64_t)p * R + i) * nth + j) * (L + 1);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int m = 2 * (4 * mt + b) + par;
          if (m > L) continue;
          T vr = re[a][b], vi = im[a][b];
          if (mid) {
            const T am = midv[par * RB + rr];
            switch (m & 3) {  // e^{-i m pi/2}
              case 0: vr += am; break;
              case 1: vi -= am; break;
              case 2: vr -= am; break;
              default: vi += am; break;
            }
          }
          Gr[m] = mk<T>(vr * dscale, vi * dscale);
        }
      }
    }
    __syncthreads();
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

template <typename T> struct ShPlan {
  int RB, S, nslab;
  bool dft_smem;
  size_t rbytes;
};

template <typename T> ShPlan<T> sh_plan(const ShTables<T>& tab) {
  // one CTA (512 threads) per SM: the deepest slab (<= 8 planes) and the largest ring batch that fit;
  // the DFT table moves to global memory (L1) only if shared memory cannot hold it
  ShPlan<T> pl;
  const size_t budget = 220 * 1024;
  for (int pass = 0; pass < 2; ++pass) {
    const bool ds = (pass == 0);
    for (int S = 8; S >= 1; --S) {
      int RB = 64;
      auto tot = [&](int rb) { return ring_layout<T>(tab.N, S, tab.nth, tab.nph, tab.R, rb, tab.Kh, tab.MP, ds).total; };
      while (RB > 8 && tot(RB) > budget) RB -= 8;
      if (tot(RB) <= budget && (RB >= 32 || S == 1)) {
        pl.S = S;
        pl.RB = RB;
        pl.dft_smem = ds;
        pl.nslab = (tab.N + S - 1) / S;
        pl.rbytes = tot(RB);
        return pl;
      }
    }
  }
  pl.S = 1;
  pl.RB = 8;
  pl.dft_smem = false;
  pl.nslab = tab.N;
  pl.rbytes = ring_layout<T>(tab.N, 1, tab.nth, tab.nph, tab.R, 8, tab.Kh, tab.MP, false).total;
  return pl;
}

}  // namespace

template <typename T> size_t sh_ring_workspace_elems(const ShTables<T>& tab) {
  return (size_t)tab.R * tab.nth * (tab.L + 1);
}

template <typename T>
cudaError_t launch_sh_analysis(const float* vols, int64_t B, const T* shifts, int shift_stride, const ShTables<T>& tab,
                               cplx_t<T>* F, cplx_t<T>* Gws, int64_t gws_particles, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const int N = tab.N, ncf = ncoef(tab.L);
  const ShPlan<T> plan = sh_plan<T>(tab);
  cudaError_t e = cudaFuncSetAttribute(k_sh_rings<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.rbytes);
  if (e != cudaSuccess) return e;
  const int JP = 8;
  const size_t lbytes = leg_layout<T>(4, JP, tab.L).total;
  const int lthreads = std::min(512, (leg_tiles(tab.L) + 31) / 32 * 32);
  e = cudaFuncSetAttribute(k_sh_legendre<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lbytes);
  if (e != cudaSuccess) return e;
  for (int64_t c0 = 0; c0 < B; c0 += gws_particles) {
    const int64_t nb = std::min<int64_t>(gws_particles, B - c0);
    k_sh_rings<T><<<(unsigned)(nb * plan.nslab), kRingThreads, plan.rbytes, st>>>(
        vols + c0 * (int64_t)N * N * N, shifts ? shifts + c0 * shift_stride : nullptr, shift_stride, tab, plan.S,
        plan.nslab, plan.RB, plan.dft_smem, Gws);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
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
