// k_newton.cu -- stage 4: evaluation of C_L, grad, Hess and the frequency-marching Newton refinement.
//
// PAPER.md: Eq. 4 with reading C1, C_L(g) = sum_l sum_{m,n} conj(M^l_mn) D^l_mn(g);
// closed-form derivatives; Newton in the Euler chart;
// Algorithm 1 lines 3-8.  Half-plane form:
//   per (m >= 0, n) and rotation:  T0 = sum_l conj(M^l_mn) d^l,  T1 = sum_l conj(M^l_mn) d'^l,
//   U = sum_l l(l+1) conj(M^l_mn) d^l,  T2 = -cot(b) T1 + q_mn T0 - U  (Wigner ODE for d''),
//   q_mn = (m^2 + n^2 - 2mn cos b)/sin^2 b;  z_k = T_k e^{-i(ma+ng)}, w = 1 (m=0) or 2:
//   C = sum w Re z0, dC/da = sum w m Im z0, dC/db = sum w Re z1, dC/dg = sum w n Im z0,
//   H_aa = -sum w m^2 Re z0, H_gg = -sum w n^2 Re z0, H_ag = -sum w mn Re z0,
//   H_ab = sum w m Im z1, H_bg = sum w n Im z1, H_bb = sum w Re z2 = sum w Re((q_mn T0 - U) e) - cot(b) dC/db.
//
// B200 mapping: one CTA per particle.  Work item = one recurrence run (RunDesc, common.cuh): the l-run of the pair
// (l0, n) also yields the Wigner d of its symmetry partner ((n, l0) or (-n, -l0)) up to a sign, so one recurrence
// feeds two pairs' sums -- half the recurrence work of a per-pair walk.  A thread keeps CG candidates' recurrence
// state in registers (each M^l load and recurrence coefficient shared by CG candidates); the candidate groups run
// concurrently on slices of the CTA; M^l streams through a per-thread cp.async ring in shared memory.  Runs are
// grouped by l0 (long runs first) and dealt boustrophedon.  Block reductions are fixed-order (deterministic: no
// atomics), one FP64 row sum per thread.  The 3x3 Newton solve runs in FP64.
#include <float.h>

#include <cstdlib>

#include "common.cuh"
#include "wigner.cuh"

namespace matcha {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxCG = 10;  // candidates per register group
constexpr int kRedStride = kThreads + 1;  // row pitch of the partial sums: a lane per row reads conflict-free
constexpr int kRing = 4;    // M^l is requested kRing degrees ahead of its use (per-thread cp.async ring in smem)

template <int BYTES> __device__ __forceinline__ void cp_async_ca(void* sdst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(sa), "l"(gsrc), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <typename T> struct CandShared {
  T cb, sb, cot, invs2;
  BetaLogs<T> bl;
};

struct SmemLayout {
  // offsets in bytes
  size_t theta, cand, ea, eg, red, ring, sums, prevc, invl, invll, flags, total;
};

template <typename T> __host__ __device__ inline SmemLayout smem_layout(int Q, int L, int cg) {
  SmemLayout s;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 15) & ~size_t(15);
    return r;
  };
  s.theta = take(sizeof(double) * 3 * Q);
  s.cand = take(sizeof(CandShared<T>) * Q);
  s.ea = take(sizeof(cplx_t<T>) * Q * (L + 1));
  s.eg = take(sizeof(cplx_t<T>) * Q * (2 * L + 1));
  s.red = take(sizeof(T) * 10 * cg * kRedStride);  // per-thread partial sums [value][thread] (padded rows)
  s.ring = take(sizeof(cplx_t<T>) * kRing * 2 * kThreads);  // per-thread cp.async ring of M^l (pairs A, B)
  s.sums = take(sizeof(double) * 10 * Q);
  s.prevc = take(sizeof(double) * Q);
  s.invl = take(sizeof(T) * (kMaxL + 2));
  s.invll = take(sizeof(T) * (kMaxL + 2));
  s.flags = take(sizeof(int) * (2 * Q + 4));
  s.total = o;
  return s;
}

__device__ __forceinline__ double wrap2pi(double x) {
  double y = fmod(x, 2.0 * kPi);
  if (y < 0) y += 2.0 * kPi;
  if (y >= 2.0 * kPi) y -= 2.0 * kPi;
  return y;
}

// chart canonicalisation (reading C15)
__device__ __forceinline__ void canon(double* e) {
  double b = wrap2pi(e[1]);
  double a = e[0], g = e[2];
  if (b > kPi) {
    b = 2.0 * kPi - b;
    a += kPi;
    g += kPi;
  }
  e[0] = wrap2pi(a);
  e[1] = b;
  e[2] = wrap2pi(g);
}

// largest eigenvalue of a symmetric 3x3 (aa,bb,gg,ab,ag,bg), closed-form trigonometric roots
__device__ double sym3_lambda_max(const double* h) {
  const double a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5];
  const double p1 = d * d + e * e + f * f;
  const double q = (a + b + c) / 3.0;
  if (p1 == 0.0) return fmax(a, fmax(b, c));
  const double p2 = (a - q) * (a - q) + (b - q) * (b - q) + (c - q) * (c - q) + 2.0 * p1;
  const double p = sqrt(p2 / 6.0);
  const double ba = (a - q) / p, bb = (b - q) / p, bc = (c - q) / p, bd = d / p, be = e / p, bf = f / p;
  double r = 0.5 * (ba * (bb * bc - bf * bf) - bd * (bd * bc - bf * be) + be * (bd * bf - bb * be));
  r = fmin(1.0, fmax(-1.0, r));
  const double phi = acos(r) / 3.0;
  return q + 2.0 * p * cos(phi);
}

// Newton step with the eigen-shift safeguard (reading C13): H_reg = H if lambda_max < 0,
// else H - (lambda_max + 1e-6 ||H||_F) I; delta = -H_reg^{-1} g  (0 if H_reg is singular)
__device__ void newton_delta(const double* g, const double* h, double* dl) {
  const double lmax = sym3_lambda_max(h);
  const double fro = sqrt(h[0] * h[0] + h[1] * h[1] + h[2] * h[2] + 2.0 * (h[3] * h[3] + h[4] * h[4] + h[5] * h[5]));
  const double sh = (lmax < 0.0) ? 0.0 : (lmax + 1e-6 * fro);
  const double a = h[0] - sh, b = h[1] - sh, c = h[2] - sh, d = h[3], e = h[4], f = h[5];
  // symmetric [[a d e][d b f][e f c]] ; adjugate
  const double c00 = b * c - f * f, c01 = e * f - d * c, c02 = d * f - b * e;
  const double c11 = a * c - e * e, c12 = d * e - a * f, c22 = a * b - d * d;
  const double det = a * c00 + d * c01 + e * c02;
  if (det == 0.0 || !isfinite(det)) {
    dl[0] = dl[1] = dl[2] = 0.0;
    return;
  }
  const double inv = 1.0 / det;
  dl[0] = -(c00 * g[0] + c01 * g[1] + c02 * g[2]) * inv;
  dl[1] = -(c01 * g[0] + c11 * g[1] + c12 * g[2]) * inv;
  dl[2] = -(c02 * g[0] + c12 * g[1] + c22 * g[2]) * inv;
}

// Prepare per-rotation shared data for candidates [0, Q): trig of beta and phase tables.
template <typename T>
__device__ void prepare_candidates(const double* theta, int Q, int L, CandShared<T>* cs, cplx_t<T>* ea,
                                   cplx_t<T>* eg) {
  for (int c = threadIdx.x; c < Q; c += blockDim.x) {
    const double b = theta[3 * c + 1];
    double sb = sin(b), cb = cos(b);
    double sbc = fmax(fabs(sb), 1e-6);  // reading C16: clamp in cot b and 1/sin^2 b
    CandShared<T> s;
    s.cb = (T)cb;
    s.sb = (T)sb;
    s.cot = (T)(cb / sbc);
    s.invs2 = (T)(1.0 / (sbc * sbc));
    s.bl = beta_logs<T>(b);
    cs[c] = s;
  }
  // e^{-i m a} (m = 0..L), e^{-i n g} (n = -L..L), phases reduced in FP64
  const int na = L + 1, ng = 2 * L + 1;
  for (int t = threadIdx.x; t < Q * (na + ng); t += blockDim.x) {
    const int c = t / (na + ng), r = t % (na + ng);
    double ph;
    if (r < na) ph = -(double)r * theta[3 * c + 0];
    else ph = -(double)(r - na - L) * theta[3 * c + 2];
    ph -= 2.0 * kPi * rint(ph * (0.5 / kPi));  // FP64 reduction to [-pi, pi] (|ph| <= 2 pi kMaxL)
    T s, co;
    if (sizeof(T) == 4) {
      float sf, cf;
      sincosf((float)ph, &sf, &cf);  // reduced argument: the accurate fast path of sincosf
      s = (T)sf;
      co = (T)cf;
    } else {
      double sd, cd;
      sincos(ph, &sd, &cd);
      s = (T)sd;
      co = (T)cd;
    }
    if (r < na) ea[c * na + r] = mk<T>(co, s);
    else eg[c * ng + (r - na)] = mk<T>(co, s);
  }
}

// Evaluate C_L (and, if DERIV, grad and Hess) at rotations [0,Q) -> sums[c][10] (FP64 in smem).
// Work item = one RunDesc: the recurrence of pair A = (l0, nA) also yields its partner B's d (up to the sign sB), so
// one set of recurrence registers feeds two pairs' sums (T0, T1, U for A and for B).  The G = ceil(Q/CG) candidate
// groups run concurrently on G slices of the CTA (Tg = kThreads/G threads each, every slice walks all runs), so the
// few long runs of a small band are not walked G times in sequence.
template <typename T, int CG, bool DERIV>
__device__ void eval_block(const cplx_t<T>* __restrict__ M, int L, int Q, const RunDesc* __restrict__ runs,
                           const T* __restrict__ run_lnc, const CandShared<T>* cs, const cplx_t<T>* ea,
                           const cplx_t<T>* eg, const T* inv_l, const T* inv_ll, T* red, cplx_t<T>* ring,
                           double* sums) {
  constexpr int NV = DERIV ? 10 : 1;
  const int nruns = run_count(L);
  const int tid = threadIdx.x;
  const int na = L + 1, ng = 2 * L + 1;
  constexpr int NVAL = NV * CG;
  const int G = (Q + CG - 1) / CG, Tg = kThreads / G;
  const int g = tid / Tg, lt = tid - g * Tg;
  T* acc = red + tid;  // this thread's partial sums: value (v, k) at acc[(v * CG + k) * kRedStride]
#pragma unroll
  for (int i = 0; i < NVAL; ++i) acc[i * kRedStride] = T(0);
  if (g < G) {
    const int c0 = g * CG;
    // candidate indices of this group (clamped: duplicates of the last are computed, then ignored)
    int cid[CG];
#pragma unroll
    for (int k = 0; k < CG; ++k) cid[k] = min(c0 + k, Q - 1);

    for (int r = 0;; ++r) {
      const int base = r * Tg;
      if (base >= nruns) break;
      const int ri = base + ((r & 1) ? (Tg - 1 - lt) : lt);
      if (ri >= nruns) continue;
      const RunDesc rd = runs[ri];
      const int m = rd.mA, n = rd.nA;
      const int l0 = m > abs(n) ? m : abs(n);
      const bool pairB = rd.mB >= 0;
      const int mB = pairB ? rd.mB : m, nB = pairB ? rd.nB : n;
      // weight of B's terms: (1 or 2) x the symmetry sign, 0 when A runs alone
      const T sB = (nB == m && ((m - n) & 1)) ? T(-1) : T(1);
      const T wB = pairB ? sB * ((mB == 0) ? T(1) : T(2)) : T(0);
      const T lnC = run_lnc[ri];
      const int mn = m * n, m2 = m * m, n2 = n * n;
      // recurrence state
      T d[CG], dprev[CG], dp[CG], dpprev[CG];
      T a0r[CG], a0i[CG], a1r[CG], a1i[CG], aur[CG], aui[CG];  // pair A: T0, T1, U
      T b0r[CG], b0i[CG], b1r[CG], b1i[CG], bur[CG], bui[CG];  // pair B
#pragma unroll
      for (int k = 0; k < CG; ++k) {
        T dd, ddp = T(0);
        wigner_seed<T, DERIV>(m, n, lnC, cs[cid[k]].bl, dd, ddp);
        d[k] = dd;
        dp[k] = ddp;
        dprev[k] = T(0);
        dpprev[k] = T(0);
        a0r[k] = a0i[k] = a1r[k] = a1i[k] = aur[k] = aui[k] = T(0);
        b0r[k] = b0i[k] = b1r[k] = b1i[k] = bur[k] = bui[k] = T(0);
      }
      T cbk[CG], sbk[CG];
#pragma unroll
      for (int k = 0; k < CG; ++k) {
        cbk[k] = cs[cid[k]].cb;
        sbk[k] = cs[cid[k]].sb;
      }
      (void)sbk;
      // M^l_mn for l = l0.. lives at half_offset(l) + m(2l+1) + n + l: consecutive degrees differ by
      // (l+1)(2l+1) + 2m + 1 (B's step is A's + 2(mB - m)).  Each thread streams its run's M^l (A and B) through
      // its own kRing-deep cp.async ring in shared memory, kRing degrees ahead of use (no registers held by the
      // loads in flight); the l-loop is unrolled by two so that d^{l-1} is overwritten in place by d^{l+1}.
      const cplx_t<T>* pA = M + rd.offA;
      const cplx_t<T>* pB = M + rd.offB;
      int inc = (l0 + 1) * (2 * l0 + 1) + 2 * m + 1;  // pointer step li -> li + 1; grows by 4 li + 5
      const int dB = 2 * (mB - m);
      int li = l0;                                     // next degree to request
      cplx_t<T>* rg = ring + tid;                      // slot (j, pair) at rg[(2 j + pair) * kThreads]
      auto request = [&](int slot) {
        if (li <= L) {
          cp_async_ca<sizeof(cplx_t<T>)>(rg + (2 * slot) * kThreads, pA);
          cp_async_ca<sizeof(cplx_t<T>)>(rg + (2 * slot + 1) * kThreads, pB);
        }
        cp_async_commit();
        pA += inc;
        pB += inc + dB;
        inc += 4 * li + 5;
        ++li;
      };
#pragma unroll
      for (int j = 0; j < kRing; ++j) request(j);
      T sq = T(0);
      auto accumulate = [&](int l, int slot, const T* dd, const T* ddp) {
        cp_async_wait<kRing - 1>();  // degree l has landed
        const cplx_t<T> Ma = rg[(2 * slot) * kThreads], Mb = rg[(2 * slot + 1) * kThreads];
        // conj(M) = (mr, -mi)
#pragma unroll
        for (int k = 0; k < CG; ++k) {
          a0r[k] = fma(Ma.x, dd[k], a0r[k]);
          a0i[k] = fma(-Ma.y, dd[k], a0i[k]);
          b0r[k] = fma(Mb.x, dd[k], b0r[k]);
          b0i[k] = fma(-Mb.y, dd[k], b0i[k]);
        }
        if (DERIV) {
          const T ll = (T)(l * (l + 1));
          const T uar = ll * Ma.x, uai = ll * Ma.y, ubr = ll * Mb.x, ubi = ll * Mb.y;
#pragma unroll
          for (int k = 0; k < CG; ++k) {
            a1r[k] = fma(Ma.x, ddp[k], a1r[k]);
            a1i[k] = fma(-Ma.y, ddp[k], a1i[k]);
            aur[k] = fma(uar, dd[k], aur[k]);
            aui[k] = fma(-uai, dd[k], aui[k]);
            b1r[k] = fma(Mb.x, ddp[k], b1r[k]);
            b1i[k] = fma(-Mb.y, ddp[k], b1i[k]);
            bur[k] = fma(ubr, dd[k], bur[k]);
            bui[k] = fma(-ubi, dd[k], bui[k]);
          }
        }
        request(slot);  // the slot is consumed (its values are in registers): degree l + kRing
      };
      // (cur, old) = (d^l, d^{l-1}) -> old := d^{l+1}:  d^{l+1} = (A cos b - B) d^l - C d^{l-1},
      //                                                 d'^{l+1} = (A cos b - B) d'^l - A sin b d^l - C d'^{l-1}
      auto advance = [&](int l, const T* cur, T* old, const T* curp, T* oldp) {
        T A, Bc, Cc;
        rec_coef<T>(l, mn, m2, n2, inv_l, inv_ll, A, Bc, Cc, sq);
#pragma unroll
        for (int k = 0; k < CG; ++k) {
          const T coef = fma(A, cbk[k], -Bc);
          if (DERIV) oldp[k] = fma(coef, curp[k], fma(-A * sbk[k], cur[k], -Cc * oldp[k]));
          old[k] = fma(coef, cur[k], -Cc * old[k]);
        }
      };
      for (int l = l0, slot = 0;; l += 2, slot = (slot + 2) & (kRing - 1)) {
        accumulate(l, slot, d, dp);
        if (l == L) break;
        advance(l, d, dprev, dp, dpprev);  // dprev := d^{l+1}
        accumulate(l + 1, slot + 1, dprev, dpprev);
        if (l + 1 == L) break;
        advance(l + 1, dprev, d, dpprev, dp);  // d := d^{l+2}
      }
      // assembly with the phase e^{-i(m a + n g)} of each pair; both pairs' terms are summed in registers before
      // the one read-modify-write of this thread's partial sums.  H_bb's -cot(b) T1 part is factored out of the sum
      // (cot is per rotation): value 5 collects w Re((q_mn T0 - U) e) and -cot dC/db is added after the reduction.
      const T wA = (m == 0) ? T(1) : T(2);
#pragma unroll
      for (int k = 0; k < CG; ++k) {
        T v[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = T(0);
        auto contrib = [&](int pm, int pn, T w, T t0r, T t0i, T t1r, T t1i, T ur, T ui) {
          const cplx_t<T> pa = ea[cid[k] * na + pm], pg = eg[cid[k] * ng + (pn + L)];
          const T er = pa.x * pg.x - pa.y * pg.y, ei = pa.x * pg.y + pa.y * pg.x;
          const T z0r = t0r * er - t0i * ei, z0i = t0r * ei + t0i * er;
          v[0] = fma(w, z0r, v[0]);
          if (DERIV) {
            const CandShared<T>& c = cs[cid[k]];
            const T fm = (T)pm, fn = (T)pn;
            const T z1r = t1r * er - t1i * ei, z1i = t1r * ei + t1i * er;
            const T qmn = ((T)(pm * pm + pn * pn) - T(2) * (T)(pm * pn) * c.cb) * c.invs2;
            const T uR = ur * er - ui * ei;
            const T wz0 = w * z0r, wz0i = w * z0i, wz1i = w * z1i;
            v[1] = fma(fm, wz0i, v[1]);
            v[2] = fma(w, z1r, v[2]);
            v[3] = fma(fn, wz0i, v[3]);
            v[4] = fma(-fm * fm, wz0, v[4]);
            v[5] = fma(w, fma(qmn, z0r, -uR), v[5]);
            v[6] = fma(-fn * fn, wz0, v[6]);
            v[7] = fma(fm, wz1i, v[7]);
            v[8] = fma(-fm * fn, wz0, v[8]);
            v[9] = fma(fn, wz1i, v[9]);
          }
        };
        contrib(m, n, wA, a0r[k], a0i[k], a1r[k], a1i[k], aur[k], aui[k]);
        contrib(mB, nB, wB, b0r[k], b0i[k], b1r[k], b1i[k], bur[k], bui[k]);
#pragma unroll
        for (int i = 0; i < NV; ++i) acc[(i * CG + k) * kRedStride] += v[i];
      }
    }
  }
  // deterministic block reduction: one thread per row (group, value) sums the group's Tg partials in a fixed order in
  // FP64 (four interleaved chains, combined in a fixed order)
  __syncthreads();
  for (int i = tid; i < G * NVAL; i += kThreads) {
    const int gg = i / NVAL, vk = i - gg * NVAL;
    const T* row = red + vk * kRedStride + gg * Tg;
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
    int t = 0;
    for (; t + 4 <= Tg; t += 4) {
#pragma unroll
      for (int q = 0; q < 4; ++q) s4[q] += (double)row[t + q];
    }
    for (; t < Tg; ++t) s4[0] += (double)row[t];
    const int v = vk / CG, k = vk % CG, c = gg * CG + k;
    if (c < Q) sums[c * 10 + v] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  }
  __syncthreads();
  if (DERIV) {
    for (int c = tid; c < Q; c += kThreads) sums[c * 10 + 5] -= (double)cs[c].cot * sums[c * 10 + 2];
    __syncthreads();
  }
}

template <typename T>
__device__ void load_inv_tables(T* inv_l, T* inv_ll) {
  for (int l = threadIdx.x; l <= kMaxL + 1; l += blockDim.x) {
    inv_l[l] = l ? (T)(1.0 / l) : T(0);
    inv_ll[l] = l ? (T)(1.0 / ((double)l * (l + 1))) : T(0);
  }
}

// ------------------------------------------------------------------ matcha_eval_corr kernel
template <typename T, int CG>
__global__ void __launch_bounds__(kThreads, (sizeof(T) == 4 && CG <= 5) ? 2 : 1) k_eval_corr(NewtonArgs<T> a, bool derivs) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.L_eval, Q = a.Q;
  const SmemLayout lay = smem_layout<T>(Q, L, CG);
  double* theta = (double*)(smem + lay.theta);
  CandShared<T>* cs = (CandShared<T>*)(smem + lay.cand);
  cplx_t<T>* ea = (cplx_t<T>*)(smem + lay.ea);
  cplx_t<T>* eg = (cplx_t<T>*)(smem + lay.eg);
  T* red = (T*)(smem + lay.red);
  cplx_t<T>* ring = (cplx_t<T>*)(smem + lay.ring);
  double* sums = (double*)(smem + lay.sums);
  T* inv_l = (T*)(smem + lay.invl);
  T* inv_ll = (T*)(smem + lay.invll);
  const int64_t p = blockIdx.x;
  const cplx_t<T>* M = a.M + p * a.strideM;
  for (int t = threadIdx.x; t < 3 * Q; t += blockDim.x) theta[t] = (double)a.euler[p * Q * 3 + t];
  load_inv_tables(inv_l, inv_ll);
  __syncthreads();
  prepare_candidates<T>(theta, Q, L, cs, ea, eg);
  __syncthreads();
  if (derivs) eval_block<T, CG, true>(M, L, Q, a.runs, a.run_lnc, cs, ea, eg, inv_l, inv_ll, red, ring, sums);
  else eval_block<T, CG, false>(M, L, Q, a.runs, a.run_lnc, cs, ea, eg, inv_l, inv_ll, red, ring, sums);
  for (int c = threadIdx.x; c < Q; c += blockDim.x) {
    const double* s = sums + c * 10;
    a.value[p * Q + c] = (T)s[0];
    if (!isfinite(s[0])) atomicOr(a.flags, FLAG_NONFINITE);
    if (derivs) {
      if (a.grad)
        for (int k = 0; k < 3; ++k) a.grad[(p * Q + c) * 3 + k] = (T)s[1 + k];
      if (a.hess)
        for (int k = 0; k < 6; ++k) a.hess[(p * Q + c) * 6 + k] = (T)s[4 + k];
    }
  }
}

// ------------------------------------------------------------------ matcha_newton_refine kernel
// One CTA per particle: all of its candidates share every read of M (ALU-bound, not HBM-bound).
template <typename T, int CG>
__global__ void __launch_bounds__(kThreads, (sizeof(T) == 4 && CG <= 5) ? 2 : 1) k_newton_refine(NewtonArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int Q = a.Q;
  const int64_t p = blockIdx.x;
  const int Lmax_b = a.bands[a.nbands - 1];
  const SmemLayout lay = smem_layout<T>(Q, Lmax_b, CG);
  double* theta = (double*)(smem + lay.theta);
  CandShared<T>* cs = (CandShared<T>*)(smem + lay.cand);
  cplx_t<T>* ea = (cplx_t<T>*)(smem + lay.ea);
  cplx_t<T>* eg = (cplx_t<T>*)(smem + lay.eg);
  T* red = (T*)(smem + lay.red);
  cplx_t<T>* ring = (cplx_t<T>*)(smem + lay.ring);
  double* sums = (double*)(smem + lay.sums);
  T* inv_l = (T*)(smem + lay.invl);
  T* inv_ll = (T*)(smem + lay.invll);
  double* prevc = (double*)(smem + lay.prevc);
  int* act = (int*)(smem + lay.flags);   // [Q] active (not padding)
  int* run = act + Q;                    // [Q] still iterating in this band
  int* any = run + Q;                    // [1]
  const cplx_t<T>* M = a.M + p * a.strideM;
  const int64_t cb0 = p * Q;             // global index of this particle's first candidate
  for (int t = threadIdx.x; t < 3 * Q; t += blockDim.x) theta[t] = (double)a.euler[cb0 * 3 + t];
  for (int c = threadIdx.x; c < Q; c += blockDim.x) act[c] = a.idx ? (a.idx[cb0 + c] >= 0) : 1;
  load_inv_tables(inv_l, inv_ll);
  __syncthreads();
  for (int j = 0; j < a.nbands; ++j) {
    const int L = a.bands[j];
    for (int c = threadIdx.x; c < Q; c += blockDim.x) run[c] = act[c];
    for (int s = 0; s < a.iters; ++s) {
      if (threadIdx.x == 0) {
        int x = 0;
        for (int c = 0; c < Q; ++c) x |= run[c];
        *any = x;
      }
      __syncthreads();
      if (!*any) break;
      prepare_candidates<T>(theta, Q, L, cs, ea, eg);
      __syncthreads();
      eval_block<T, CG, true>(M, L, Q, a.runs, a.run_lnc, cs, ea, eg, inv_l, inv_ll, red, ring, sums);
      for (int c = threadIdx.x; c < Q; c += blockDim.x) {
        if (!run[c]) continue;
        const double* sm = sums + c * 10;
        bool fin = true;
        for (int k = 0; k < 10; ++k) fin = fin && isfinite(sm[k]);
        if (!fin) {
          atomicOr(a.flags, FLAG_NONFINITE);
          run[c] = 0;
          continue;
        }
        const double C = sm[0];
        const double gn = sqrt(sm[1] * sm[1] + sm[2] * sm[2] + sm[3] * sm[3]);
        if (a.tol_grad > 0 && gn < a.tol_grad * fabs(C)) { run[c] = 0; continue; }
        if (s > 0 && a.tol_obj > 0 && fabs(C - prevc[c]) < a.tol_obj * fabs(C)) { run[c] = 0; continue; }
        prevc[c] = C;
        double dl[3];
        newton_delta(sm + 1, sm + 4, dl);
        double* th = theta + 3 * c;
        th[0] += dl[0];
        th[1] += dl[1];
        th[2] += dl[2];
        canon(th);
        const double dn = sqrt(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
        if (a.tol_step > 0 && dn < a.tol_step) run[c] = 0;
      }
      __syncthreads();
    }
  }
  // final C_{L_J} of every candidate and the argmax
  prepare_candidates<T>(theta, Q, Lmax_b, cs, ea, eg);
  __syncthreads();
  // value only: twice the candidates per thread (no derivative state): half the walks of the runs
  if (sizeof(T) == 4 && CG == 5 && Q > CG && Q <= 2 * CG)
    eval_block<T, 2 * CG, false>(M, Lmax_b, Q, a.runs, a.run_lnc, cs, ea, eg, inv_l, inv_ll, red, ring, sums);
  else if (sizeof(T) == 4 && CG == 4 && Q > CG)
    eval_block<T, 2 * CG, false>(M, Lmax_b, Q, a.runs, a.run_lnc, cs, ea, eg, inv_l, inv_ll, red, ring, sums);
  else
    eval_block<T, CG, false>(M, Lmax_b, Q, a.runs, a.run_lnc, cs, ea, eg, inv_l, inv_ll, red, ring, sums);
  for (int t = threadIdx.x; t < 3 * Q; t += blockDim.x) a.euler[cb0 * 3 + t] = (T)theta[t];
  for (int c = threadIdx.x; c < Q; c += blockDim.x) {
    const double v = act[c] ? sums[c * 10] : -INFINITY;
    a.score[cb0 + c] = (T)v;
    if (act[c] && !isfinite(v)) atomicOr(a.flags, FLAG_NONFINITE);
  }
  if (threadIdx.x == 0) {
    int b = -1;
    double bv = -INFINITY;
    for (int c = 0; c < Q; ++c)
      if (act[c] && (b < 0 || sums[c * 10] > bv)) {
        b = c;
        bv = sums[c * 10];
      }
    a.best[p] = b;
  }
}

template <typename T, int CG> cudaError_t launch_eval_cg(const NewtonArgs<T>& a, bool derivs, cudaStream_t s) {
  const SmemLayout lay = smem_layout<T>(a.Q, a.L_eval, CG);
  cudaError_t e = cudaFuncSetAttribute(k_eval_corr<T, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.total);
  if (e != cudaSuccess) return e;
  k_eval_corr<T, CG><<<(unsigned)a.B, kThreads, lay.total, s>>>(a, derivs);
  return cudaGetLastError();
}

template <typename T, int CG> cudaError_t launch_newton_cg(const NewtonArgs<T>& a, cudaStream_t s) {
  const SmemLayout lay = smem_layout<T>(a.Q, a.bands[a.nbands - 1], CG);
  cudaError_t e =
      cudaFuncSetAttribute(k_newton_refine<T, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.total);
  if (e != cudaSuccess) return e;
  k_newton_refine<T, CG><<<(unsigned)a.B, kThreads, lay.total, s>>>(a);
  return cudaGetLastError();
}

// candidate-group size: registers hold 10*CG recurrence values and 10*CG accumulators per thread
template <typename T> int pick_cg(int Q) {
  if (sizeof(T) == 8) return Q >= 2 ? 2 : 1;
  if (Q <= 2) return Q;
  if (Q <= 4) return 4;
  if (Q % 5 == 0 || Q == 9) return 5;
  return 4;
}

}  // namespace

template <typename T> cudaError_t launch_eval_corr(const NewtonArgs<T>& a, bool derivs, cudaStream_t s) {
  if (a.B == 0 || a.Q == 0) return cudaSuccess;
  switch (pick_cg<T>(a.Q)) {
    case 1: return launch_eval_cg<T, 1>(a, derivs, s);
    case 2: return launch_eval_cg<T, 2>(a, derivs, s);
    case 4: return launch_eval_cg<T, 4>(a, derivs, s);
    default: return launch_eval_cg<T, 5>(a, derivs, s);
  }
}

template <typename T> cudaError_t launch_newton_refine(const NewtonArgs<T>& a, cudaStream_t s) {
  if (a.B == 0 || a.Q == 0) return cudaSuccess;
  switch (pick_cg<T>(a.Q)) {
    case 1: return launch_newton_cg<T, 1>(a, s);
    case 2: return launch_newton_cg<T, 2>(a, s);
    case 4: return launch_newton_cg<T, 4>(a, s);
    default: return launch_newton_cg<T, 5>(a, s);
  }
}

template cudaError_t launch_eval_corr<float>(const NewtonArgs<float>&, bool, cudaStream_t);
template cudaError_t launch_eval_corr<double>(const NewtonArgs<double>&, bool, cudaStream_t);
template cudaError_t launch_newton_refine<float>(const NewtonArgs<float>&, cudaStream_t);
template cudaError_t launch_newton_refine<double>(const NewtonArgs<double>&, cudaStream_t);

// SURVEY f4 ("evaluate alignment against multiple candidate templates"): the best template per particle
// reading C29: templates are compared by C_{L_J} / ||H_{<=L_J}||_w (the raw inner product grows with the template's
// energy; the particle's norm is common to all templates); ties -> lowest template index
template <typename T>
__global__ void k_select_template(const T* __restrict__ cand, const double* __restrict__ tnorm, int nt, int64_t B,
                                  bool keep_shift, T* poses, int pstride, int* __restrict__ tsel) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B) return;
  int k = 0;
  double bv = (double)cand[b * 8 + 6] / tnorm[0];
  for (int t = 1; t < nt; ++t) {
    const double v = (double)cand[((int64_t)t * B + b) * 8 + 6] / tnorm[t];
    if (v > bv) {
      bv = v;
      k = t;
    }
  }
  const T* c = cand + ((int64_t)k * B + b) * 8;
  T* o = poses + b * pstride;
  for (int q = 0; q < 8; ++q)
    if (!(keep_shift && q >= 3 && q <= 5)) o[q] = c[q];
  if (pstride >= 9) o[8] = (T)k;
  if (tsel) tsel[b] = k;
}

template <typename T>
cudaError_t launch_select_template(const T* cand, const double* tnorm, int nt, int64_t B, bool keep_shift, T* poses,
                                   int pstride, int* tsel, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  k_select_template<T><<<(unsigned)((B + 127) / 128), 128, 0, s>>>(cand, tnorm, nt, B, keep_shift, poses, pstride,
                                                                    tsel);
  return cudaGetLastError();
}
template cudaError_t launch_select_template<float>(const float*, const double*, int, int64_t, bool, float*, int, int*,
                                                   cudaStream_t);
template cudaError_t launch_select_template<double>(const double*, const double*, int, int64_t, bool, double*, int,
                                                    int*, cudaStream_t);

// ||H_k||_w over l <= L for templates k < nt (one CTA each, fixed-order FP64 block reduction)
template <typename T>
__global__ void __launch_bounds__(256) k_template_norms(const cplx_t<T>* __restrict__ H, int Lmax, int L, int R,
                                                        double* __restrict__ out) {
  __shared__ double red[256];
  const cplx_t<T>* h = H + (int64_t)blockIdx.x * ncoef(Lmax) * R;
  double e = 0;
  for (int t = threadIdx.x; t < ncoef(L) * R; t += blockDim.x) {
    const int lm = t / R, i = t - lm * R;
    int l = 0;
    while ((l + 1) * (l + 2) / 2 <= lm) ++l;
    const int m = lm - l * (l + 1) / 2;
    const double r = i + 0.5;
    const cplx_t<T> v = h[t];
    e += (m ? 2.0 : 1.0) * r * r * ((double)v.x * v.x + (double)v.y * v.y);  // |h_{l,-m}| = |h_{l,m}|
  }
  red[threadIdx.x] = e;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sqrt(red[0]);
}

template <typename T>
cudaError_t launch_template_norms(const cplx_t<T>* H, int nt, int Lmax, int L, int R, double* out, cudaStream_t s) {
  k_template_norms<T><<<(unsigned)nt, 256, 0, s>>>(H, Lmax, L, R, out);
  return cudaGetLastError();
}
template cudaError_t launch_template_norms<float>(const float2*, int, int, int, int, double*, cudaStream_t);
template cudaError_t launch_template_norms<double>(const double2*, int, int, int, int, double*, cudaStream_t);

// poses[b] = {alpha, beta, gamma, (shift untouched), score, best}
template <typename T>
__global__ void k_gather_poses(const T* euler, const T* score, const int32_t* best, int64_t B, int Q, bool zero_shift,
                               T* poses) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int k = best[b];
  T* o = poses + b * 8;
  if (k >= 0) {
    o[0] = euler[(b * Q + k) * 3 + 0];
    o[1] = euler[(b * Q + k) * 3 + 1];
    o[2] = euler[(b * Q + k) * 3 + 2];
    o[6] = score[b * Q + k];
  } else {
    o[0] = o[1] = o[2] = T(0);
    o[6] = -INFINITY;
  }
  if (zero_shift) o[3] = o[4] = o[5] = T(0);
  o[7] = (T)k;
}

template <typename T>
cudaError_t launch_gather_poses(const T* euler, const T* score, const int32_t* best, int64_t B, int Q, bool zero_shift,
                                T* poses, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  k_gather_poses<T><<<(unsigned)((B + 127) / 128), 128, 0, s>>>(euler, score, best, B, Q, zero_shift, poses);
  return cudaGetLastError();
}
template cudaError_t launch_gather_poses<float>(const float*, const float*, const int32_t*, int64_t, int, bool,
                                                float*, cudaStream_t);
template cudaError_t launch_gather_poses<double>(const double*, const double*, const int32_t*, int64_t, int, bool,
                                                 double*, cudaStream_t);

}  // namespace matcha
