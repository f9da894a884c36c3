// k_search.cu -- stage 3: coarse exhaustive SO(3) search of C_{L0} and top-N_C local maxima.
//
// north_star stage (3); PAPER.md P:147-151 (SOFFT grid of O((K L0)^3) points, N_C strongest local maxima),
// Algorithm 1 lines 1-2; readings C9 (grid), C10-C11 (local maxima, ties, padding).
// Per beta slice j:
//   X_{j,mn} = sum_{l=max(m,|n|)}^{L0} conj(M^l_mn) d^l_mn(beta_j)       (Wigner-d contraction)
//   C(alpha_a, beta_j, gamma_c) = Re Y_{0,c} + 2 Re sum_{m>=1} Y_{m,c} e^{-i m alpha_a},
//   Y_{m,c} = sum_n X_{j,mn} e^{-i n gamma_c}                             (separable 2-D DFT, Hermitian X)
//
// B200 mapping: one CTA per particle.  When the grid fits in shared memory (L0 <= 9 at K = 2) k_so3_grid keeps it
// resident and runs each phase over the whole grid (few barriers); otherwise k_so3_search (below) streams it:  M(l <= L0) is staged in shared memory (4 KiB at L0 = 8); d is
// produced on the fly by the l-recurrence (no table traffic); the grid is never materialised: a rolling
// 3-slice window in shared memory feeds the 26-neighbour test of slice j-1 while slice j is computed, so
// L0 = 12 (70k nodes, 275 KiB) needs no cluster.  Maxima go to a shared list; the N_C winners are chosen
// by an order-independent block arg-max on (score desc, index asc) -- deterministic.
#include <cstdlib>

#include "common.cuh"
#include "wigner.cuh"

namespace matcha {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kCap = 2048;

struct SearchLayout {
  size_t Ms, X, Y, sl, tmv, tmi, mxv, mxi, tw, cs, cs_idx, invl, invll, misc, beta, red_s, red_i, total;
};

template <typename T> __host__ __device__ inline SearchLayout search_layout(int L0, int K) {
  const int nb = K * (L0 + 1), na = 2 * K * (L0 + 1);
  SearchLayout s;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t r = o;
    o += (b + 15) & ~size_t(15);
    return r;
  };
  s.Ms = take(sizeof(cplx_t<T>) * half_size(L0));
  s.X = take(sizeof(cplx_t<T>) * (L0 + 1) * (2 * L0 + 1));
  s.Y = take(sizeof(cplx_t<T>) * (L0 + 1) * na);
  s.sl = take(sizeof(T) * na * na);             // raw C values of the current beta slice
  s.tmv = take(sizeof(T) * na * na);            // gamma-pass of the 3x3 (alpha,gamma) max filter
  s.tmi = take(sizeof(int) * na * na);
  s.mxv = take(sizeof(T) * 3 * na * na);        // rolling 3-slice window of the in-slice 3x3 maxima
  s.mxi = take(sizeof(int) * 3 * na * na);
  s.tw = take(sizeof(cplx_t<T>) * na);
  s.cs = take(sizeof(T) * kCap);
  s.cs_idx = take(sizeof(int) * kCap);
  s.invl = take(sizeof(T) * (kMaxL + 2));
  s.invll = take(sizeof(T) * (kMaxL + 2));
  s.misc = take(sizeof(T) * 8 + sizeof(int) * 8);
  s.beta = take(sizeof(T) * 3 * nb);           // per slice: cos beta_j, ln cos(beta_j/2), ln sin(beta_j/2)
  s.red_s = take(sizeof(T) * kWarps);
  s.red_i = take(sizeof(int) * kWarps);
  s.total = o;
  return s;
}

// key order: (score desc, index asc); returns true if (s1,i1) ranks before (s2,i2)
template <typename T> __device__ __forceinline__ bool before(T s1, int i1, T s2, int i2) {
  return s1 > s2 || (s1 == s2 && i1 < i2);
}

// t / d for 0 <= t < 2^32 / d^2 (d <= 128 here): multiply-high by ceil(2^32 / d), no integer division
__device__ __forceinline__ int fdiv(int t, uint32_t magic) { return (int)__umulhi((uint32_t)t, magic); }

template <typename T>
__global__ void __launch_bounds__(kThreads) k_so3_search(SearchArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L0 = a.L0, K = a.K;
  const int nb = K * (L0 + 1), na = 2 * K * (L0 + 1), ng = na;
  const SearchLayout lay = search_layout<T>(L0, K);
  cplx_t<T>* Ms = (cplx_t<T>*)(smem + lay.Ms);
  cplx_t<T>* X = (cplx_t<T>*)(smem + lay.X);
  cplx_t<T>* Y = (cplx_t<T>*)(smem + lay.Y);
  T* sl = (T*)(smem + lay.sl);
  T* tmv = (T*)(smem + lay.tmv);
  int* tmi = (int*)(smem + lay.tmi);
  T* mxv = (T*)(smem + lay.mxv);
  int* mxi = (int*)(smem + lay.mxi);
  cplx_t<T>* tw = (cplx_t<T>*)(smem + lay.tw);
  T* cs = (T*)(smem + lay.cs);
  int* ci = (int*)(smem + lay.cs_idx);
  T* inv_l = (T*)(smem + lay.invl);
  T* inv_ll = (T*)(smem + lay.invll);
  int* cnt = (int*)(smem + lay.misc + sizeof(T) * 8);
  T* bsl = (T*)(smem + lay.beta);  // [3][nb]
  const uint32_t mg = (uint32_t)((0x100000000ull + ng - 1) / ng);  // fdiv magic for ng
  T* red_s = (T*)(smem + lay.red_s);
  int* red_i = (int*)(smem + lay.red_i);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t p = blockIdx.x;

  const cplx_t<T>* Mp = a.M + p * a.strideM;
  for (int t = tid; t < half_size(L0); t += kThreads) Ms[t] = Mp[t];
  for (int t = tid; t < na; t += kThreads) {
    double s, c;
    sincospi(2.0 * t / na, &s, &c);
    tw[t] = mk<T>((T)c, (T)(-s));  // e^{-2 pi i t/na}
  }
  for (int l = tid; l <= kMaxL + 1; l += kThreads) {
    inv_l[l] = l ? (T)(1.0 / l) : T(0);
    inv_ll[l] = l ? (T)(1.0 / ((double)l * (l + 1))) : T(0);
  }
  for (int j = tid; j < nb; j += kThreads) {
    const double beta = (j + 0.5) * kPi / nb;
    const BetaLogs<T> bl = beta_logs<T>(beta);
    bsl[j] = (T)cos(beta);
    bsl[nb + j] = bl.lnc;
    bsl[2 * nb + j] = bl.lns;
  }
  if (tid == 0) *cnt = 0;
  __syncthreads();

  const int npairs = pair_count(L0);
  const int w0 = 2 * L0 + 1;
  // Local maxima by a separable max filter on the unique keys (score desc, index asc): node p is a strict local
  // maximum over its 26 neighbours iff it is the best key of its closed 3x3x3 neighbourhood.
  auto test_slice = [&](int jj) {
    for (int t = tid; t < na * ng; t += kThreads) {
      const int ip = jj * na * ng + t;
      T bv = mxv[(jj % 3) * na * ng + t];
      int bi = mxi[(jj % 3) * na * ng + t];
      if (jj > 0) {
        const T v = mxv[((jj - 1) % 3) * na * ng + t];
        const int i = mxi[((jj - 1) % 3) * na * ng + t];
        if (before(v, i, bv, bi)) {
          bv = v;
          bi = i;
        }
      }
      if (jj + 1 < nb) {
        const T v = mxv[((jj + 1) % 3) * na * ng + t];
        const int i = mxi[((jj + 1) % 3) * na * ng + t];
        if (before(v, i, bv, bi)) {
          bv = v;
          bi = i;
        }
      }
      if (bi == ip) {
        const int slot = atomicAdd(cnt, 1);
        if (slot < kCap) {
          cs[slot] = bv;
          ci[slot] = ip;
        } else {
          atomicOr(a.flags, FLAG_OVERFLOW);
        }
      }
    }
  };
  // in-slice 3x3 (alpha, gamma periodic) max of the keys of slice j -> window slot j % 3
  auto filter_slice = [&](int j) {
    for (int t = tid; t < na * ng; t += kThreads) {
      const int aa = fdiv(t, mg), c = t - aa * ng;
      const int cm = c == 0 ? ng - 1 : c - 1, cp = c == ng - 1 ? 0 : c + 1;
      const int base = j * na * ng + aa * ng;
      T bv = sl[t];
      int bi = base + c;
      const T v1 = sl[aa * ng + cm], v2 = sl[aa * ng + cp];
      if (before(v1, base + cm, bv, bi)) {
        bv = v1;
        bi = base + cm;
      }
      if (before(v2, base + cp, bv, bi)) {
        bv = v2;
        bi = base + cp;
      }
      tmv[t] = bv;
      tmi[t] = bi;
    }
    __syncthreads();
    T* ov = mxv + (j % 3) * na * ng;
    int* oi = mxi + (j % 3) * na * ng;
    for (int t = tid; t < na * ng; t += kThreads) {
      const int aa = fdiv(t, mg), c = t - aa * ng;
      const int am = aa == 0 ? na - 1 : aa - 1, ap = aa == na - 1 ? 0 : aa + 1;
      T bv = tmv[t];
      int bi = tmi[t];
      const T v1 = tmv[am * ng + c], v2 = tmv[ap * ng + c];
      const int i1 = tmi[am * ng + c], i2 = tmi[ap * ng + c];
      if (before(v1, i1, bv, bi)) {
        bv = v1;
        bi = i1;
      }
      if (before(v2, i2, bv, bi)) {
        bv = v2;
        bi = i2;
      }
      ov[t] = bv;
      oi[t] = bi;
    }
  };

  for (int j = 0; j < nb; ++j) {
    const T cb = bsl[j];
    BetaLogs<T> bl;
    bl.lnc = bsl[nb + j];
    bl.lns = bsl[2 * nb + j];
    // X_{j,mn}
    for (int pi = tid; pi < npairs; pi += kThreads) {
      const PairDesc pd = a.pairs[pi];
      const int m = pd.m, n = pd.n, l0 = max(m, abs(n));
      T d, dd, dprev = T(0), sq = T(0);
      wigner_seed<T, false>(m, n, a.pair_lnc[pi], bl, d, dd);
      T xr = T(0), xi = T(0);
      int off = pd.off0;
      for (int l = l0;; ++l) {
        const cplx_t<T> Ml = Ms[off];
        xr = fma(Ml.x, d, xr);
        xi = fma(-Ml.y, d, xi);
        if (l == L0) break;
        T A, Bc, Cc;
        rec_coef<T>(l, m * n, m * m, n * n, inv_l, inv_ll, A, Bc, Cc, sq);
        const T dn = fma(A * d, cb, -fma(Bc, d, Cc * dprev));
        dprev = d;
        d = dn;
        off += (l + 1) * (2 * l + 1) + 2 * m + 1;
      }
      X[m * w0 + (n + L0)] = mk<T>(xr, xi);
    }
    __syncthreads();
    // Y_{m,c} = sum_n X_mn e^{-i n gamma_c}
    for (int t = tid; t < (L0 + 1) * ng; t += kThreads) {
      const int m = fdiv(t, mg), c = t - m * ng;
      T yr = T(0), yi = T(0);
      int k = (ng - (L0 * c) % ng) % ng;  // (n c) mod ng at n = -L0, then + c per step
      for (int n = -L0; n <= L0; ++n) {
        const cplx_t<T> x = X[m * w0 + (n + L0)];
        const cplx_t<T> e = tw[k];
        k += c;
        if (k >= ng) k -= ng;
        yr = fma(x.x, e.x, fma(-x.y, e.y, yr));
        yi = fma(x.x, e.y, fma(x.y, e.x, yi));
      }
      Y[m * ng + c] = mk<T>(yr, yi);
    }
    __syncthreads();
    // C(alpha_a, beta_j, gamma_c)
    T* cur = sl;
    for (int t = tid; t < na * ng; t += kThreads) {
      const int aa = fdiv(t, mg), c = t - aa * ng;
      T s = Y[c].x;
      T s2 = T(0);
      int k = 0;
      for (int m = 1; m <= L0; ++m) {
        k += aa;
        if (k >= na) k -= na;
        const cplx_t<T> y = Y[m * ng + c], e = tw[k];
        s2 = fma(y.x, e.x, fma(-y.y, e.y, s2));
      }
      cur[t] = fma(T(2), s2, s);
    }
    __syncthreads();
    filter_slice(j);
    __syncthreads();
    if (j >= 1) test_slice(j - 1);
  }
  test_slice(nb - 1);
  __syncthreads();

  // top-N_C selection by (score desc, index asc)
  const int total = min(*cnt, kCap);
  for (int k = 0; k < a.ncand; ++k) {
    T bs = -INFINITY;
    int bi = 0x7fffffff;
    for (int t = tid; t < total; t += kThreads)
      if (ci[t] >= 0 && before(cs[t], ci[t], bs, bi)) {
        bs = cs[t];
        bi = ci[t];
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const T s2 = __shfl_xor_sync(0xffffffffu, bs, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (before(s2, i2, bs, bi)) {
        bs = s2;
        bi = i2;
      }
    }
    if (lane == 0) {
      red_s[warp] = bs;
      red_i[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      T s = red_s[0];
      int i = red_i[0];
      for (int w = 1; w < kWarps; ++w)
        if (before(red_s[w], red_i[w], s, i)) {
          s = red_s[w];
          i = red_i[w];
        }
      const int64_t o = p * a.ncand + k;
      if (i != 0x7fffffff) {
        const int c = i % ng, aa = (i / ng) % na, jj = i / (ng * na);
        a.euler[o * 3 + 0] = (T)(2.0 * kPi * aa / na);
        a.euler[o * 3 + 1] = (T)((jj + 0.5) * kPi / nb);
        a.euler[o * 3 + 2] = (T)(2.0 * kPi * c / ng);
        a.score[o] = s;
        a.idx[o] = i;
        for (int t = 0; t < total; ++t)
          if (ci[t] == i) ci[t] = -1;  // taken
      } else {
        a.euler[o * 3 + 0] = a.euler[o * 3 + 1] = a.euler[o * 3 + 2] = T(0);
        a.score[o] = -INFINITY;
        a.idx[o] = -1;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ full-grid variant (grid resident in smem)
// Used when the whole (beta, alpha, gamma) grid of C_{L0} fits in shared memory (L0 <= 9 at K = 2): every phase is
// data-parallel over the whole grid, so the CTA passes ~6 barriers instead of ~5 per beta slice.
//   phase 1  X[j][m][n] for all slices: one item = (pair, kJG slices) sharing the recurrence coefficients
//   phase 2  Y[j][m][c] = sum_n X e^{-i n gamma_c}          (per chunk of jc slices)
//   phase 3  C[j][a][c] = Re Y[j][0][c] + 2 Re sum_m Y e^{-i m alpha_a}   (4 alphas per item, Y loads shared)
//   phase 4  strict 26-neighbour maxima by direct comparison of keys (score desc, index asc), early exit
//   phase 5  top-N_C by one warp: N_C rounds of a warp arg-max over the candidate list (deterministic)
constexpr int kGThreads = 512;
constexpr int kJG = 4;

struct GridLayout {
  size_t Ms, ea, eg, beta, invl, invll, X, Y, C, cs, ci, misc, total;
};

template <typename T> __host__ __device__ inline GridLayout grid_layout(int L0, int K, int jc) {
  const int nb = K * (L0 + 1), na = 2 * K * (L0 + 1), nm = L0 + 1, w0 = 2 * L0 + 1;
  GridLayout s;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t r = o;
    o += (b + 15) & ~size_t(15);
    return r;
  };
  s.Ms = take(sizeof(cplx_t<T>) * half_size(L0));
  s.ea = take(sizeof(cplx_t<T>) * nm * na);  // e^{-i m alpha_a}
  s.eg = take(sizeof(cplx_t<T>) * w0 * na);  // e^{-i n gamma_c}, n = -L0..L0
  s.beta = take(sizeof(T) * 3 * nb);
  s.invl = take(sizeof(T) * (L0 + 2));
  s.invll = take(sizeof(T) * (L0 + 2));
  s.X = take(sizeof(cplx_t<T>) * (size_t)nb * nm * w0);
  s.Y = take(sizeof(cplx_t<T>) * (size_t)jc * nm * na);
  s.C = take(sizeof(T) * (size_t)nb * (na + 2) * (na + 2));  // one-node periodic halo in alpha and gamma
  s.cs = take(sizeof(T) * kCap);
  s.ci = take(sizeof(int) * kCap);
  s.misc = take(sizeof(int) * 4);
  s.total = o;
  return s;
}

// L0C, KC: compile-time L0 and oversampling (0 = runtime) -- with both fixed every grid index is a constant expression
template <typename T, int L0C, int KC>
__global__ void __launch_bounds__(kGThreads) k_so3_grid(SearchArgs<T> a, int jc) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L0 = L0C ? L0C : a.L0, K = KC ? KC : a.K;
  const int nb = K * (L0 + 1), na = 2 * K * (L0 + 1), ng = na, nm = L0 + 1, w0 = 2 * L0 + 1;
  const GridLayout lay = grid_layout<T>(L0, K, jc);
  cplx_t<T>* Ms = (cplx_t<T>*)(smem + lay.Ms);
  cplx_t<T>* Ea = (cplx_t<T>*)(smem + lay.ea);
  cplx_t<T>* Eg = (cplx_t<T>*)(smem + lay.eg);
  T* bsl = (T*)(smem + lay.beta);  // [3][nb]: cos beta_j, ln cos(beta_j/2), ln sin(beta_j/2)
  T* inv_l = (T*)(smem + lay.invl);
  T* inv_ll = (T*)(smem + lay.invll);
  cplx_t<T>* X = (cplx_t<T>*)(smem + lay.X);
  cplx_t<T>* Y = (cplx_t<T>*)(smem + lay.Y);
  T* C = (T*)(smem + lay.C);
  T* cs = (T*)(smem + lay.cs);
  int* ci = (int*)(smem + lay.ci);
  int* cnt = (int*)(smem + lay.misc);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t p = blockIdx.x;

  const cplx_t<T>* Mp = a.M + p * a.strideM;
  for (int t = tid; t < half_size(L0); t += kGThreads) Ms[t] = Mp[t];
  // phase tables e^{-2 pi i k/na} at k = (m a) mod na and (n c) mod ng (exact integer reduction)
  for (int t = tid; t < (nm + w0) * na; t += kGThreads) {
    const int r = t / na, c = t - r * na;
    const int f = r < nm ? r : r - nm - L0;  // m, or n
    const int k = ((f * c) % na + na) % na;
    double sn, cn;
    sincospi(2.0 * k / na, &sn, &cn);
    const cplx_t<T> e = mk<T>((T)cn, (T)(-sn));
    if (r < nm) Ea[c * nm + r] = e;             // Ea[a][m] = e^{-i m alpha_a}
    else Eg[c * w0 + (r - nm)] = e;             // Eg[c][n + L0] = e^{-i n gamma_c}
  }
  for (int l = tid; l <= L0 + 1; l += kGThreads) {
    inv_l[l] = l ? (T)(1.0 / l) : T(0);
    inv_ll[l] = l ? (T)(1.0 / ((double)l * (l + 1))) : T(0);
  }
  for (int j = tid; j < nb; j += kGThreads) {
    const double beta = (j + 0.5) * kPi / nb;
    const BetaLogs<T> bl = beta_logs<T>(beta);
    bsl[j] = (T)cos(beta);
    bsl[nb + j] = bl.lnc;
    bsl[2 * nb + j] = bl.lns;
  }
  if (tid == 0) *cnt = 0;
  __syncthreads();

  // phase 1: X_{j,mn} = sum_l conj(M^l_mn) d^l_mn(beta_j)
  const int npairs = pair_count(L0), njg = (nb + kJG - 1) / kJG;
  for (int it = tid; it < npairs * njg; it += kGThreads) {
    const int pi = it % npairs, jg = it / npairs;
    const PairDesc pd = a.pairs[pi];
    const int m = pd.m, n = pd.n, l0 = max(m, abs(n));
    const T lnC = a.pair_lnc[pi];
    T d[kJG], dprev[kJG], xr[kJG], xi[kJG], cb[kJG];
#pragma unroll
    for (int q = 0; q < kJG; ++q) {
      const int j = min(jg * kJG + q, nb - 1);
      BetaLogs<T> bl;
      bl.lnc = bsl[nb + j];
      bl.lns = bsl[2 * nb + j];
      T dd;
      wigner_seed<T, false>(m, n, lnC, bl, d[q], dd);
      cb[q] = bsl[j];
      dprev[q] = xr[q] = xi[q] = T(0);
    }
    int off = pd.off0;
    T sq = T(0);
    for (int l = l0;; ++l) {
      const cplx_t<T> Ml = Ms[off];
#pragma unroll
      for (int q = 0; q < kJG; ++q) {
        xr[q] = fma(Ml.x, d[q], xr[q]);
        xi[q] = fma(-Ml.y, d[q], xi[q]);
      }
      if (l == L0) break;
      T A, Bc, Cc;
      rec_coef<T>(l, m * n, m * m, n * n, inv_l, inv_ll, A, Bc, Cc, sq);
#pragma unroll
      for (int q = 0; q < kJG; ++q) {
        const T dn = fma(A * d[q], cb[q], -fma(Bc, d[q], Cc * dprev[q]));
        dprev[q] = d[q];
        d[q] = dn;
      }
      off += (l + 1) * (2 * l + 1) + 2 * m + 1;
    }
#pragma unroll
    for (int q = 0; q < kJG; ++q) {
      const int j = jg * kJG + q;
      if (j < nb) X[((size_t)j * nm + m) * w0 + (n + L0)] = mk<T>(xr[q], xi[q]);
    }
  }
  __syncthreads();

  const int PA = na + 2, PG = ng + 2, PP = PA * PG;  // padded grid: [nb][PA][PG]
  const int naq = (PA + 3) / 4;
  const uint32_t mgn = (uint32_t)((0x100000000ull + ng - 1) / ng), mgq = (uint32_t)((0x100000000ull + naq - 1) / naq);
  const uint32_t mgp = (uint32_t)((0x100000000ull + PG - 1) / PG);
  for (int j0 = 0; j0 < nb; j0 += jc) {
    const int nj = min(jc, nb - j0);
    // phase 2: Y_{m,c} = sum_n X_mn e^{-i n gamma_c}
    for (int t = tid; t < nj * nm * ng; t += kGThreads) {
      const int r = fdiv(t, mgn), c = t - r * ng;  // r = jj * nm + m
      const cplx_t<T>* x = X + ((size_t)j0 * nm + r) * w0;
      const cplx_t<T>* eg = Eg + c * w0;
      T yr = T(0), yi = T(0);
#pragma unroll
      for (int n = 0; n < w0; ++n) {
        const cplx_t<T> xv = x[n];
        const cplx_t<T> e = eg[n];
        yr = fma(xv.x, e.x, fma(-xv.y, e.y, yr));
        yi = fma(xv.x, e.y, fma(xv.y, e.x, yi));
      }
      Y[t] = mk<T>(yr, yi);
    }
    __syncthreads();
    // phase 3: C(alpha_a, beta_j, gamma_c) on the halo-padded grid (padded index a_p = a + 1, c_p = c + 1, wrapped),
    // four alphas per item sharing the Y loads
    for (int t = tid; t < nj * naq * PG; t += kGThreads) {
      const int r = fdiv(t, mgp), cp = t - r * PG, jj = fdiv(r, mgq), aq = r - jj * naq;
      const int c = cp == 0 ? ng - 1 : (cp > ng ? 0 : cp - 1);
      const cplx_t<T>* y = Y + (size_t)jj * nm * ng + c;
      int av[4];
      T s2[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int ap = min(4 * aq + q, PA - 1);
        av[q] = ap == 0 ? na - 1 : (ap > na ? 0 : ap - 1);
        s2[q] = T(0);
      }
      const T s0 = y[0].x;
      const cplx_t<T>* eq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) eq[q] = Ea + av[q] * nm;
#pragma unroll
      for (int m = 1; m <= L0; ++m) {
        const cplx_t<T> yy = y[m * ng];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const cplx_t<T> e = eq[q][m];
          s2[q] = fma(yy.x, e.x, fma(-yy.y, e.y, s2[q]));
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (4 * aq + q < PA) C[(size_t)(j0 + jj) * PP + (4 * aq + q) * PG + cp] = fma(T(2), s2[q], s0);
    }
    __syncthreads();
  }

  // phase 4: strict local maxima (26 neighbours; alpha, gamma periodic, beta clamped).  Every point first meets its
  // 8 in-slice neighbours at constant offsets of the padded grid (branch-free; the exact key order is only needed on
  // a value tie); the few survivors of a warp are then tested against their 18 neighbours in slices j +- 1 by 18
  // lanes at once (one ballot per survivor).
  const uint32_t mg_ng = (uint32_t)((0x100000000ull + ng - 1) / ng), mg_na = (uint32_t)((0x100000000ull + na - 1) / na);
  const int ntot = nb * na * ng;
  auto key_index = [&](int j, int ap, int cp) {  // logical node index of a padded position
    const int a2 = ap == 0 ? na - 1 : (ap > na ? 0 : ap - 1);
    const int c2 = cp == 0 ? ng - 1 : (cp > ng ? 0 : cp - 1);
    return (j * na + a2) * ng + c2;
  };
  for (int base = 0; base < ntot; base += kGThreads) {
    const int ip = base + tid;
    const bool valid = ip < ntot;
    const int ipc = valid ? ip : ntot - 1;
    const int r = fdiv(ipc, mg_ng), c = ipc - r * ng, j = fdiv(r, mg_na), aa = r - j * na;
    const T* cc = C + (size_t)j * PP + (aa + 1) * PG + (c + 1);
    const T v = cc[0];
    const T nv[8] = {cc[-PG - 1], cc[-PG], cc[-PG + 1], cc[-1], cc[1], cc[PG - 1], cc[PG], cc[PG + 1]};
    bool gt = true, eq = false;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      gt = gt && (v > nv[q]);
      eq = eq || (v == nv[q]);
    }
    bool surv = valid && gt;
    if (valid && eq) {  // value tie: exact key order (score desc, index asc)
      surv = true;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int qq = q < 4 ? q : q + 1;
        const int iq = key_index(j, aa + 1 + qq / 3 - 1, c + 1 + qq % 3 - 1);
        surv = surv && before(v, ipc, nv[q], iq);
      }
    }
    unsigned bal = __ballot_sync(0xffffffffu, surv);
    while (bal) {
      const int src = __ffs(bal) - 1;
      bal &= bal - 1;
      const int ipx = __shfl_sync(0xffffffffu, ipc, src);
      const T vx = __shfl_sync(0xffffffffu, v, src);
      const int rx = fdiv(ipx, mg_ng), cx = ipx - rx * ng, jx = fdiv(rx, mg_na), ax = rx - jx * na;
      bool ok = true;
      if (lane < 18) {
        const int jn = jx + (lane < 9 ? -1 : 1), q = lane < 9 ? lane : lane - 9;
        if (jn >= 0 && jn < nb) {
          const int ap = ax + q / 3, cp = cx + q % 3;  // padded: (ax + 1) + (q / 3 - 1)
          ok = before(vx, ipx, C[(size_t)jn * PP + ap * PG + cp], key_index(jn, ap, cp));
        }
      }
      if (__all_sync(0xffffffffu, ok) && lane == src) {
        const int slot = atomicAdd(cnt, 1);
        if (slot < kCap) {
          cs[slot] = vx;
          ci[slot] = ipx;
        } else {
          atomicOr(a.flags, FLAG_OVERFLOW);
        }
      }
    }
  }
  __syncthreads();

  // phase 5: top-N_C by (score desc, index asc), one warp
  if (warp == 0) {
    const int total = min(*cnt, kCap);
    for (int k = 0; k < a.ncand; ++k) {
      T bs = -INFINITY;
      int bi = 0x7fffffff, bt = -1;
      for (int t = lane; t < total; t += 32)
        if (ci[t] >= 0 && before(cs[t], ci[t], bs, bi)) {
          bs = cs[t];
          bi = ci[t];
          bt = t;
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const T s2 = __shfl_xor_sync(0xffffffffu, bs, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        const int t2 = __shfl_xor_sync(0xffffffffu, bt, o);
        if (before(s2, i2, bs, bi)) {
          bs = s2;
          bi = i2;
          bt = t2;
        }
      }
      if (lane == 0) {
        const int64_t o = p * a.ncand + k;
        if (bi != 0x7fffffff) {
          const int c = bi % ng, aa = (bi / ng) % na, jj = bi / (ng * na);
          a.euler[o * 3 + 0] = (T)(2.0 * kPi * aa / na);
          a.euler[o * 3 + 1] = (T)((jj + 0.5) * kPi / nb);
          a.euler[o * 3 + 2] = (T)(2.0 * kPi * c / ng);
          a.score[o] = bs;
          a.idx[o] = bi;
          ci[bt] = -1;  // taken
        } else {
          a.euler[o * 3 + 0] = a.euler[o * 3 + 1] = a.euler[o * 3 + 2] = T(0);
          a.score[o] = -INFINITY;
          a.idx[o] = -1;
        }
      }
      __syncwarp();
    }
  }
}


// ------------------------------------------------------------------ large grids (L0 = 30, K = 2)
// The paper's operating point has a 62 x 124 x 124 grid (953k nodes, 3.8 MB per particle in FP32):
// no CTA can hold it, so the search runs in three passes over a global grid workspace:
//   k_so3_slice     one CTA per (beta slice, particle): X (M read through L1/L2), Y, C as in k_so3_search; C -> grid
//   k_so3_slice_max one CTA per (beta slice, particle): strict 26-neighbour maxima of slice j by the key order
//                   (score desc, index asc), the slice's best n_cand written to a [slice][n_cand] list
//   k_so3_merge     one CTA per particle: the n_cand best of the nb * n_cand slice winners (deterministic)
// The global top-n_cand of the local maxima is contained in the union of the per-slice top-n_cand lists.
constexpr int kBThreads = 256;
constexpr int kSliceCap = 3072;

template <typename T>
__global__ void __launch_bounds__(kBThreads) k_so3_slice(SearchArgs<T> a, T* __restrict__ grid) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L0 = a.L0, K = a.K, nb = K * (L0 + 1), na = 2 * K * (L0 + 1), ng = na, w0 = 2 * L0 + 1;
  cplx_t<T>* X = reinterpret_cast<cplx_t<T>*>(smem);     // [L0+1][2L0+1]
  cplx_t<T>* Y = X + (L0 + 1) * w0;                       // [L0+1][ng]
  cplx_t<T>* tw = Y + (L0 + 1) * ng;                      // [na]
  T* inv_l = reinterpret_cast<T*>(tw + na);               // [kMaxL+2]
  T* inv_ll = inv_l + kMaxL + 2;
  const int j = blockIdx.x, tid = threadIdx.x;
  const int64_t p = blockIdx.y;
  const cplx_t<T>* Mp = a.M + p * a.strideM;
  for (int t = tid; t < na; t += kBThreads) {
    double sn, cs;
    sincospi(2.0 * t / na, &sn, &cs);
    tw[t] = mk<T>((T)cs, (T)(-sn));  // e^{-2 pi i t/na}
  }
  for (int l = tid; l <= kMaxL + 1; l += kBThreads) {
    inv_l[l] = l ? (T)(1.0 / l) : T(0);
    inv_ll[l] = l ? (T)(1.0 / ((double)l * (l + 1))) : T(0);
  }
  const double beta = (j + 0.5) * kPi / nb;
  const BetaLogs<T> bl = beta_logs<T>(beta);
  const T cb = (T)cos(beta);
  __syncthreads();
  for (int pi = tid; pi < pair_count(L0); pi += kBThreads) {
    const PairDesc pd = a.pairs[pi];
    const int m = pd.m, n = pd.n, l0 = max(m, abs(n));
    T d, dd, dprev = T(0), sq = T(0);
    wigner_seed<T, false>(m, n, a.pair_lnc[pi], bl, d, dd);
    T xr = T(0), xi = T(0);
    int off = pd.off0;
    for (int l = l0;; ++l) {
      const cplx_t<T> Ml = Mp[off];
      xr = fma(Ml.x, d, xr);
      xi = fma(-Ml.y, d, xi);
      if (l == L0) break;
      T A, Bc, Cc;
      rec_coef<T>(l, m * n, m * m, n * n, inv_l, inv_ll, A, Bc, Cc, sq);
      const T dn = fma(A * d, cb, -fma(Bc, d, Cc * dprev));
      dprev = d;
      d = dn;
      off += (l + 1) * (2 * l + 1) + 2 * m + 1;
    }
    X[m * w0 + (n + L0)] = mk<T>(xr, xi);
  }
  __syncthreads();
  for (int t = tid; t < (L0 + 1) * ng; t += kBThreads) {
    const int m = t / ng, c = t - m * ng;
    T yr = T(0), yi = T(0);
    int k = (ng - (L0 * c) % ng) % ng;  // (n c) mod ng at n = -L0, then + c per step
    for (int n = -L0; n <= L0; ++n) {
      const cplx_t<T> x = X[m * w0 + (n + L0)], e = tw[k];
      k += c;
      if (k >= ng) k -= ng;
      yr = fma(x.x, e.x, fma(-x.y, e.y, yr));
      yi = fma(x.x, e.y, fma(x.y, e.x, yi));
    }
    Y[m * ng + c] = mk<T>(yr, yi);
  }
  __syncthreads();
  T* out = grid + (p * nb + j) * (int64_t)na * ng;
  for (int t = tid; t < na * ng; t += kBThreads) {
    const int aa = t / ng, c = t - aa * ng;
    T s2 = T(0);
    int k = 0;
    for (int m = 1; m <= L0; ++m) {
      k += aa;
      if (k >= na) k -= na;
      const cplx_t<T> y = Y[m * ng + c], e = tw[k];
      s2 = fma(y.x, e.x, fma(-y.y, e.y, s2));
    }
    out[t] = fma(T(2), s2, Y[c].x);
  }
}

template <typename T>
__global__ void __launch_bounds__(kBThreads) k_so3_slice_max(SearchArgs<T> a, const T* __restrict__ grid,
                                                             T* __restrict__ lval, int* __restrict__ lidx) {
  __shared__ T cs[kSliceCap];
  __shared__ int ci[kSliceCap];
  __shared__ int cnt;
  __shared__ T red_s[kBThreads / 32];
  __shared__ int red_i[kBThreads / 32];
  const int L0 = a.L0, K = a.K, nb = K * (L0 + 1), na = 2 * K * (L0 + 1), ng = na;
  const int j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t p = blockIdx.y;
  const T* g = grid + p * (int64_t)nb * na * ng;
  if (tid == 0) cnt = 0;
  __syncthreads();
  for (int t = tid; t < na * ng; t += kBThreads) {
    const int aa = t / ng, c = t - aa * ng;
    const int ip = j * na * ng + t;
    const T v = g[ip];
    bool mx = true;
    for (int dj = -1; dj <= 1 && mx; ++dj) {
      const int jj = j + dj;
      if (jj < 0 || jj >= nb) continue;
      for (int da = -1; da <= 1 && mx; ++da) {
        const int a2 = aa + da < 0 ? na - 1 : (aa + da >= na ? 0 : aa + da);
        for (int dc = -1; dc <= 1; ++dc) {
          if (!dj && !da && !dc) continue;
          const int c2 = c + dc < 0 ? ng - 1 : (c + dc >= ng ? 0 : c + dc);
          const int iq = (jj * na + a2) * ng + c2;
          if (iq == ip) continue;
          if (!before(v, ip, g[iq], iq)) {
            mx = false;
            break;
          }
        }
      }
    }
    if (mx) {
      const int slot = atomicAdd(&cnt, 1);
      if (slot < kSliceCap) {
        cs[slot] = v;
        ci[slot] = ip;
      } else {
        atomicOr(a.flags, FLAG_OVERFLOW);
      }
    }
  }
  __syncthreads();
  const int total = min(cnt, kSliceCap);
  for (int k = 0; k < a.ncand; ++k) {
    T bs = -INFINITY;
    int bi = 0x7fffffff;
    for (int t = tid; t < total; t += kBThreads)
      if (ci[t] >= 0 && before(cs[t], ci[t], bs, bi)) {
        bs = cs[t];
        bi = ci[t];
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const T s2 = __shfl_xor_sync(0xffffffffu, bs, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (before(s2, i2, bs, bi)) {
        bs = s2;
        bi = i2;
      }
    }
    if (lane == 0) {
      red_s[warp] = bs;
      red_i[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      T s = red_s[0];
      int i = red_i[0];
      for (int w = 1; w < kBThreads / 32; ++w)
        if (before(red_s[w], red_i[w], s, i)) {
          s = red_s[w];
          i = red_i[w];
        }
      const int64_t o = (p * nb + j) * a.ncand + k;
      lval[o] = s;
      lidx[o] = (i == 0x7fffffff) ? -1 : i;
      for (int t = 0; t < total; ++t)
        if (ci[t] == i) ci[t] = -1;  // taken
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(kBThreads) k_so3_merge(SearchArgs<T> a, const T* __restrict__ lval,
                                                         const int* __restrict__ lidx) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L0 = a.L0, K = a.K, nb = K * (L0 + 1), na = 2 * K * (L0 + 1), ng = na;
  const int n = nb * a.ncand, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* cs = reinterpret_cast<T*>(smem);
  int* ci = reinterpret_cast<int*>(cs + n);
  __shared__ T red_s[kBThreads / 32];
  __shared__ int red_i[kBThreads / 32];
  const int64_t p = blockIdx.x;
  for (int t = tid; t < n; t += kBThreads) {
    cs[t] = lval[p * n + t];
    ci[t] = lidx[p * n + t];
  }
  __syncthreads();
  for (int k = 0; k < a.ncand; ++k) {
    T bs = -INFINITY;
    int bi = 0x7fffffff;
    for (int t = tid; t < n; t += kBThreads)
      if (ci[t] >= 0 && before(cs[t], ci[t], bs, bi)) {
        bs = cs[t];
        bi = ci[t];
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const T s2 = __shfl_xor_sync(0xffffffffu, bs, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (before(s2, i2, bs, bi)) {
        bs = s2;
        bi = i2;
      }
    }
    if (lane == 0) {
      red_s[warp] = bs;
      red_i[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      T s = red_s[0];
      int i = red_i[0];
      for (int w = 1; w < kBThreads / 32; ++w)
        if (before(red_s[w], red_i[w], s, i)) {
          s = red_s[w];
          i = red_i[w];
        }
      const int64_t o = p * a.ncand + k;
      if (i != 0x7fffffff) {
        const int c = i % ng, aa = (i / ng) % na, jj = i / (ng * na);
        a.euler[o * 3 + 0] = (T)(2.0 * kPi * aa / na);
        a.euler[o * 3 + 1] = (T)((jj + 0.5) * kPi / nb);
        a.euler[o * 3 + 2] = (T)(2.0 * kPi * c / ng);
        a.score[o] = s;
        a.idx[o] = i;
        for (int t = 0; t < n; ++t)
          if (ci[t] == i) ci[t] = -1;
      } else {
        a.euler[o * 3 + 0] = a.euler[o * 3 + 1] = a.euler[o * 3 + 2] = T(0);
        a.score[o] = -INFINITY;
        a.idx[o] = -1;
      }
    }
    __syncthreads();
  }
}

// slices per Y chunk for the full-grid kernel (0 = the grid does not fit: use the rolling-window kernel)
template <typename T> int grid_chunk(int L0, int K) {
  const int nb = K * (L0 + 1);
  for (int jc = nb; jc >= 1; --jc)
    if (grid_layout<T>(L0, K, jc).total <= 225 * 1024) return jc;
  return 0;
}

}  // namespace

size_t so3_large_workspace_bytes(int L0, int K, int ncand, bool fp64) {
  const size_t nb = (size_t)K * (L0 + 1), na = 2 * (size_t)K * (L0 + 1), rs = fp64 ? 8 : 4;
  return rs * nb * na * na + nb * ncand * (rs + sizeof(int)) + 64;
}

bool so3_large_needed(int L0, int K, bool fp64) {
  return search_smem_bytes(L0, K, fp64) > 220 * 1024;
}

template <typename T> cudaError_t launch_so3_search_large(const SearchArgs<T>& a, void* ws, cudaStream_t s) {
  if (a.B == 0) return cudaSuccess;
  const int nb = a.K * (a.L0 + 1), na = 2 * a.K * (a.L0 + 1);
  if (a.L0 > kMaxL || (int64_t)nb * na * na >= (1ll << 31)) return cudaErrorInvalidValue;
  const size_t per = so3_large_workspace_bytes(a.L0, a.K, a.ncand, sizeof(T) == 8);
  T* grid = reinterpret_cast<T*>(ws);
  T* lval = grid + a.B * (int64_t)nb * na * na;
  int* lidx = reinterpret_cast<int*>(lval + a.B * (int64_t)nb * a.ncand);
  (void)per;
  const size_t s1 = sizeof(cplx_t<T>) * ((size_t)(a.L0 + 1) * (2 * a.L0 + 1) + (size_t)(a.L0 + 1) * na + na) +
                    2 * sizeof(T) * (kMaxL + 2);
  cudaError_t e = cudaFuncSetAttribute(k_so3_slice<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
  if (e != cudaSuccess) return e;
  k_so3_slice<T><<<dim3((unsigned)nb, (unsigned)a.B), kBThreads, s1, s>>>(a, grid);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_so3_slice_max<T><<<dim3((unsigned)nb, (unsigned)a.B), kBThreads, 0, s>>>(a, grid, lval, lidx);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const size_t s3 = (sizeof(T) + sizeof(int)) * (size_t)nb * a.ncand;
  e = cudaFuncSetAttribute(k_so3_merge<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s3);
  if (e != cudaSuccess) return e;
  k_so3_merge<T><<<(unsigned)a.B, kBThreads, s3, s>>>(a, lval, lidx);
  return cudaGetLastError();
}
template cudaError_t launch_so3_search_large<float>(const SearchArgs<float>&, void*, cudaStream_t);
template cudaError_t launch_so3_search_large<double>(const SearchArgs<double>&, void*, cudaStream_t);

template <typename T> cudaError_t launch_so3_search(const SearchArgs<T>& a, cudaStream_t s) {
  if (a.B == 0) return cudaSuccess;
  const int jc = grid_chunk<T>(a.L0, a.K);
  if (jc > 0) {
    const size_t bytes = grid_layout<T>(a.L0, a.K, jc).total;
    auto kern = (a.L0 == 8 && a.K == 2) ? k_so3_grid<T, 8, 2> : (a.L0 == 4 && a.K == 2) ? k_so3_grid<T, 4, 2>
                                                                                           : k_so3_grid<T, 0, 0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)a.B, kGThreads, bytes, s>>>(a, jc);
    return cudaGetLastError();
  }
  const size_t bytes = search_layout<T>(a.L0, a.K).total;
  cudaError_t e = cudaFuncSetAttribute(k_so3_search<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  k_so3_search<T><<<(unsigned)a.B, kThreads, bytes, s>>>(a);
  return cudaGetLastError();
}

template cudaError_t launch_so3_search<float>(const SearchArgs<float>&, cudaStream_t);
template cudaError_t launch_so3_search<double>(const SearchArgs<double>&, cudaStream_t);

size_t search_smem_bytes(int L0, int K, bool fp64) {
  const int jc = fp64 ? grid_chunk<double>(L0, K) : grid_chunk<float>(L0, K);
  if (jc > 0) return fp64 ? grid_layout<double>(L0, K, jc).total : grid_layout<float>(L0, K, jc).total;
  return fp64 ? search_layout<double>(L0, K).total : search_layout<float>(L0, K).total;
}

}  // namespace matcha
