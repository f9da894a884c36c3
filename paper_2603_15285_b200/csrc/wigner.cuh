// wigner.cuh -- Wigner small-d by the three-term recurrence in l at fixed (m, n) (device side).
//
// D^l_mn(a,b,g) = e^{-ima} d^l_mn(b) e^{-ing}  (App. A.3).
// For fixed (m >= 0, n) and l0 = max(m, |n|):
//   seed   d^{l0}_mn = sgn sqrt(C(2 l0, p)) cos(b/2)^p sin(b/2)^q,  p = |m+n|, q = |m-n|,
//          sgn = (-1)^(m-n) if m >= n else +1   (closed form of Wigner's sum at l = l0);
//   step   d^{l+1} = A_l cos(b) d^l - B_l d^l - C_l d^{l-1},
//          A_l = (l+1)(2l+1)/sqrt(Q_{l+1}), B_l = A_l mn/(l(l+1)), C_l = (l+1) sqrt(Q_l)/(l sqrt(Q_{l+1})),
//          Q_l = (l^2 - m^2)(l^2 - n^2)  (so C_{l0} = 0);
//   d'     differentiates the step: d'^{l+1} = A_l (cos b d'^l - sin b d^l) - B_l d'^l - C_l d'^{l-1}.
// The closed-form gradient/Hessian of C_L is assembled from these
// in k_newton.cu.  The FP64 oracle uses a different algorithm (Jacobi closed form + ladder).
#pragma once

#include "common.cuh"

namespace matcha {

template <typename T> __device__ __forceinline__ T rsqrt_t(T x);
// x >= 1 here (Q_{l+1} is a positive integer): the approximate reciprocal square root without the denormal fix-up
template <> __device__ __forceinline__ float rsqrt_t<float>(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
template <> __device__ __forceinline__ double rsqrt_t<double>(double x) { return rsqrt(x); }

template <typename T> __device__ __forceinline__ T exp_t(T x);
template <> __device__ __forceinline__ float exp_t<float>(float x) { return expf(x); }
template <> __device__ __forceinline__ double exp_t<double>(double x) { return exp(x); }

// Per-rotation quantities used by the seeds: ln cos(b/2), ln sin(b/2) (clamped away from -inf).
template <typename T> struct BetaLogs {
  T lnc, lns;  // ln cos(b/2), ln sin(b/2)
  T cs, sc;    // cos(b/2)/sin(b/2), sin(b/2)/cos(b/2) (clamped), for the seed derivative
};
template <typename T> __device__ __forceinline__ BetaLogs<T> beta_logs(double beta) {
  double c = cos(0.5 * beta), s = sin(0.5 * beta);
  BetaLogs<T> r;
  r.lnc = (T)log(fmax(c, 1e-300));
  r.lns = (T)log(fmax(s, 1e-300));
  r.cs = (T)(c / fmax(s, 1e-30));
  r.sc = (T)(s / fmax(c, 1e-30));
  return r;
}

// seed value (and beta-derivative) of d^{l0}_{mn}; lnC = 1/2 ln C(2 l0, |m+n|)
template <typename T, bool DERIV>
__device__ __forceinline__ void wigner_seed(int m, int n, T lnC, const BetaLogs<T>& bl, T& d, T& dp) {
  const int p = abs(m + n), q = abs(m - n);
  const T sgn = (m >= n && ((m - n) & 1)) ? T(-1) : T(1);
  const T ep = p ? (T)p * bl.lnc : T(0);
  const T eq = q ? (T)q * bl.lns : T(0);
  d = sgn * exp_t<T>(lnC + ep + eq);
  if (DERIV) {
    // d/db [c^p s^q] = 1/2 c^p s^q (q c/s - p s/c),  c = cos(b/2), s = sin(b/2)
    dp = T(0.5) * d * ((T)q * bl.cs - (T)p * bl.sc);
  }
}

// recurrence coefficients for the step l -> l+1.  sq: in sqrt(Q_l), out sqrt(Q_{l+1}).
// inv_l[l] = 1/l (0 at l = 0), inv_ll[l] = 1/(l(l+1)) (0 at l = 0), in shared memory.
template <typename T>
__device__ __forceinline__ void rec_coef(int l, int mn, int m2, int n2, const T* inv_l, const T* inv_ll, T& A, T& Bc,
                                         T& C, T& sq) {
  const int l1 = l + 1, l1s = l1 * l1;
  const T Q1 = (T)((l1s - m2) * (l1s - n2));
  const T rq = rsqrt_t<T>(Q1);
  A = (T)(l1 * (2 * l + 1)) * rq;
  Bc = A * (T)mn * inv_ll[l];
  C = (T)l1 * sq * rq * inv_l[l];
  sq = Q1 * rq;
}

}  // namespace matcha
