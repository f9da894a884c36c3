/*
 * oracle.cpp -- FP64 CPU ORACLE for the Matcha hot path (arXiv 2603.15285).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2603_15285_b200/) never links, imports or calls it, and this file shares no
 * code, header, table or constant generator with the CUDA sources.
 *
 * Plain, slow, obviously-correct: every step is the paper's definition written out
 * (or, for the iterative parts, the paper's algorithm in the paper's order), in double
 * precision, with the readings of SURVEY.md 8(c) (listed in DESIGN.md "Readings").
 * Citations: P:n = /root/reference/PAPER.md line n (section / equation named beside it).
 *
 * Independent algorithms relative to the GPU path:
 *   - Wigner d from the Jacobi-polynomial closed form (not the normalised l-recurrence);
 *   - d/dbeta and d2/dbeta2 by the ladder identity (not the recurrence derivative + ODE);
 *   - naive O(n_phi * L) DFT per ring (no real-data folding);
 *   - the coarse grid by DIRECT evaluation of C_{L0} at every node (no 2-D DFT);
 *   - 3x3 eigenvalues by cyclic Jacobi rotations (not closed-form trigonometric roots);
 *   - the translation correlation by a direct windowed sum over x (no FFT).
 *
 * Parity-unpinned parts (only GPU-vs-oracle parity checks them): noisy-landscape Newton
 * paths, noise aliasing in stage 1, parabolic-subpixel bias on noisy peaks.
 * translation_upsampled is pinned by: c~ at integer points = the direct circular correlation, the
 * separable contraction = the full triple sum at arbitrary points, planted fractional shifts recovered to 1/kappa.
 */
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

using cd = std::complex<double>;
using std::vector;

namespace {

const double PI = 3.14159265358979323846264338327950288;

inline int ncoef(int L) { return (L + 1) * (L + 2) / 2; }
inline int lm_index(int l, int m) { return l * (l + 1) / 2 + m; }
/* full-plane block offset: sum_{l'<l} (2l'+1)^2 */
inline long full_offset(int l) { return (long)l * (2L * l - 1) * (2L * l + 1) / 3; }
inline long full_size(int L) { return full_offset(L + 1); }

/* ---------------- rotations: ZYZ Euler chart, Eq. (3) P:79-95 ---------------- */
void matmul3(const double* A, const double* B, double* C) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += A[3 * i + k] * B[3 * k + j];
      C[3 * i + j] = s;
    }
}
void rot_z(double t, double* R) {
  double c = std::cos(t), s = std::sin(t);
  double M[9] = {c, -s, 0, s, c, 0, 0, 0, 1};
  std::memcpy(R, M, sizeof(M));
}
void rot_y(double t, double* R) {
  double c = std::cos(t), s = std::sin(t);
  double M[9] = {c, 0, s, 0, 1, 0, -s, 0, c};
  std::memcpy(R, M, sizeof(M));
}
/* g(alpha,beta,gamma) = r_z(alpha) r_y(beta) r_z(gamma)   (Eq. 3) */
void euler_to_matrix(const double* e, double* R) {
  double A[9], B[9], C[9], T[9];
  rot_z(e[0], A);
  rot_y(e[1], B);
  rot_z(e[2], C);
  matmul3(A, B, T);
  matmul3(T, C, R);
}
/* inverse chart map, reading C7 (gimbal: gamma = 0) */
void matrix_to_euler(const double* R, double* e) {
  double r33 = std::max(-1.0, std::min(1.0, R[8]));
  double b = std::acos(r33);
  double a, g;
  double sb = std::sqrt(std::max(0.0, 1.0 - r33 * r33));
  if (sb > 1e-12) {
    a = std::atan2(R[5], R[2]);
    g = std::atan2(R[7], -R[6]);
  } else if (r33 > 0) {
    a = std::atan2(R[3], R[0]);
    g = 0;
  } else {
    a = std::atan2(-R[3], -R[0]);
    g = 0;
  }
  e[0] = a; e[1] = b; e[2] = g;
}
double wrap2pi(double x) {
  double y = std::fmod(x, 2 * PI);
  if (y < 0) y += 2 * PI;
  if (y >= 2 * PI) y -= 2 * PI;
  return y;
}
/* chart canonicalisation, reading C15: beta reduced mod 2pi; beta>pi => (a+pi, 2pi-b, g+pi);
   then alpha, gamma wrapped to [0,2pi).  Uses r_y(-b) = r_z(pi) r_y(b) r_z(pi). */
void canon(double* e) {
  double b = wrap2pi(e[1]);
  double a = e[0], g = e[2];
  if (b > PI) {
    b = 2 * PI - b;
    a += PI;
    g += PI;
  }
  e[0] = wrap2pi(a);
  e[1] = b;
  e[2] = wrap2pi(g);
}

/* ---------------- Gauss-Legendre nodes (reading C4) ---------------- */
void gauss_legendre(int n, vector<double>& x, vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double z = std::cos(PI * (i + 0.75) / (n + 0.5));
    double dp = 0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (n == 1) { p1 = z; p0 = 1.0; }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (n == 1) { p1 = z; p0 = 1.0; }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
    }
    x[n - 1 - i] = z; /* ascending */
    w[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

/* ------- orthonormal associated Legendre with Condon-Shortley phase (reading C3) -------
   Y_lm(theta,phi) = P_lm(cos theta) e^{i m phi}, P_lm = sqrt((2l+1)/4pi (l-m)!/(l+m)!) P_l^m,
   P_l^m including (-1)^m.  Output P[l(l+1)/2+m], 0<=m<=l<=L. */
void legendre_norm(int L, double x, vector<double>& P) {
  P.assign(ncoef(L), 0.0);
  double s = std::sqrt(std::max(0.0, 1.0 - x * x));
  double pmm = 1.0 / std::sqrt(4 * PI);
  for (int m = 0; m <= L; ++m) {
    if (m > 0) pmm = -std::sqrt((2.0 * m + 1.0) / (2.0 * m)) * s * pmm;
    P[lm_index(m, m)] = pmm;
    if (m + 1 <= L) P[lm_index(m + 1, m)] = std::sqrt(2.0 * m + 3.0) * x * pmm;
    for (int l = m + 2; l <= L; ++l) {
      double a = std::sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)m * m));
      double b = std::sqrt((((double)(l - 1) * (l - 1)) - (double)m * m) / (4.0 * (l - 1) * (l - 1) - 1.0));
      P[lm_index(l, m)] = a * (x * P[lm_index(l - 1, m)] - b * P[lm_index(l - 2, m)]);
    }
  }
}

/* ---------------- Wigner small d, App. A.3 ----------------
   d^l_{mn}(beta) by the Jacobi-polynomial closed form of Wigner's finite sum:
   with k = l - max(|m|,|n|), a = |m-n|, b = |m+n|:
     d^l_{mn} = (-1)^lam sqrt(C(2l-k, k+a)/C(k+b, b)) sin(b/2)^a cos(b/2)^b P_k^{(a,b)}(cos beta)
   (lam = m-n when the minimum defining k is l+n or l-m, else 0).  Convention (reading C7):
   d^1_{10} = -sin(beta)/sqrt(2), d^1_{00} = cos(beta).  Output d[l][(m+l)(2l+1)+(n+l)]. */
double lbinom(int n, int k) { return std::lgamma(n + 1.0) - std::lgamma(k + 1.0) - std::lgamma(n - k + 1.0); }

void wigner_d_all(int L, double beta, vector<vector<double>>& d) {
  d.assign(L + 1, vector<double>());
  for (int l = 0; l <= L; ++l) d[l].assign((2 * l + 1) * (2 * l + 1), 0.0);
  const double x = std::cos(beta);
  const double ls = std::log(std::fabs(std::sin(0.5 * beta)));
  const double lc = std::log(std::fabs(std::cos(0.5 * beta)));
  for (int m = -L; m <= L; ++m)
    for (int n = -L; n <= L; ++n) {
      const int l0 = std::max(std::abs(m), std::abs(n));
      const int a = std::abs(m - n), b = std::abs(m + n);
      /* which of (l+n, l-n, l+m, l-m) attains the minimum at every l >= l0 */
      int lam;
      if (-n == l0) lam = m - n;       /* k = l+n */
      else if (n == l0) lam = 0;       /* k = l-n */
      else if (-m == l0) lam = 0;      /* k = l+m */
      else lam = m - n;                /* k = l-m */
      const double sgn = (lam % 2 == 0) ? 1.0 : -1.0;
      double pk_2 = 0, pk_1 = 0;
      for (int k = 0; k <= L - l0; ++k) {
        /* Jacobi P_k^{(a,b)}(x): standard three-term recurrence in the degree k */
        double pk;
        if (k == 0) pk = 1.0;
        else if (k == 1) pk = (a + 1.0) + (a + b + 2.0) * (x - 1.0) / 2.0;
        else {
          double kk = k, A = a, B = b;
          double c1 = 2.0 * kk * (kk + A + B) * (2.0 * kk + A + B - 2.0);
          double c2 = (2.0 * kk + A + B - 1.0) * ((2.0 * kk + A + B) * (2.0 * kk + A + B - 2.0) * x + A * A - B * B);
          double c3 = 2.0 * (kk + A - 1.0) * (kk + B - 1.0) * (2.0 * kk + A + B);
          pk = (c2 * pk_1 - c3 * pk_2) / c1;
        }
        pk_2 = pk_1;
        pk_1 = pk;
        const int l = l0 + k;
        double lpre = 0.5 * (lbinom(2 * l - k, k + a) - lbinom(k + b, b));
        double powpart;
        /* sin^a cos^b with 0^0 = 1 */
        double lg = lpre + (a > 0 ? a * ls : 0.0) + (b > 0 ? b * lc : 0.0);
        powpart = std::exp(lg);
        if ((a > 0 && std::sin(0.5 * beta) == 0.0) || (b > 0 && std::cos(0.5 * beta) == 0.0)) powpart = 0.0;
        if (std::sin(0.5 * beta) < 0 && (a % 2 == 1)) powpart = -powpart;
        if (std::cos(0.5 * beta) < 0 && (b % 2 == 1)) powpart = -powpart;
        d[l][(m + l) * (2 * l + 1) + (n + l)] = sgn * powpart * pk;
      }
    }
}

/* ladder identity (the "finite combination of shifted d's" of P:1295):
   d/dbeta d^l_{mn} = 1/2 [ sqrt((l+n)(l-n+1)) d^l_{m,n-1} - sqrt((l-n)(l+n+1)) d^l_{m,n+1} ] */
void ladder(int l, const vector<double>& d, vector<double>& out) {
  const int w = 2 * l + 1;
  out.assign(w * w, 0.0);
  for (int m = -l; m <= l; ++m)
    for (int n = -l; n <= l; ++n) {
      double v = 0;
      if (n - 1 >= -l) v += std::sqrt((double)(l + n) * (l - n + 1)) * d[(m + l) * w + (n - 1 + l)];
      if (n + 1 <= l) v -= std::sqrt((double)(l - n) * (l + n + 1)) * d[(m + l) * w + (n + 1 + l)];
      out[(m + l) * w + (n + l)] = 0.5 * v;
    }
}

/* ---------------- stage 1: shell SH analysis (north_star (1)) -------
   f_lm(r_i) = sum_j W_j sum_k (2pi/n_phi) u(c + r_i w_jk) conj(Y_lm(theta_j, phi_k))
   r_i = i - 1/2 (i = 1..R = N/2), n_theta = L_q+1 Gauss-Legendre nodes, n_phi = 2 L_q + 2,
   L_q = qover * L (readings C2, C4).  F layout: complex [ncoef(L)][R]. */
struct VolSampler {
  const float* v;
  int N;
  double val(int x, int y, int z) const {
    if (x < 0 || y < 0 || z < 0 || x >= N || y >= N || z >= N) return 0.0;
    return (double)v[((size_t)z * N + y) * N + x];
  }
  /* trilinear interpolation of the zero-extended volume v[z][y][x] (reading C5) */
  double operator()(double px, double py, double pz) const {
    double fx0 = std::floor(px), fy0 = std::floor(py), fz0 = std::floor(pz);
    int x0 = (int)fx0, y0 = (int)fy0, z0 = (int)fz0;
    double fx = px - fx0, fy = py - fy0, fz = pz - fz0;
    double s = 0;
    for (int dz = 0; dz < 2; ++dz)
      for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
          double w = (dx ? fx : 1 - fx) * (dy ? fy : 1 - fy) * (dz ? fz : 1 - fz);
          s += w * val(x0 + dx, y0 + dy, z0 + dz);
        }
    return s;
  }
};

/* analytic polynomial u(y) = sum coef y_x^a y_y^b y_z^c at y = R^T (p - c) (for pins) */
struct PolySampler {
  const double* terms;
  int nterms;
  double R[9];
  double cx, cy, cz;
  double operator()(double px, double py, double pz) const {
    double y0 = px - cx, y1 = py - cy, y2 = pz - cz;
    double q0 = R[0] * y0 + R[3] * y1 + R[6] * y2; /* R^T y */
    double q1 = R[1] * y0 + R[4] * y1 + R[7] * y2;
    double q2 = R[2] * y0 + R[5] * y1 + R[8] * y2;
    double s = 0;
    for (int t = 0; t < nterms; ++t) {
      const double* tm = terms + 4 * t;
      s += tm[0] * std::pow(q0, (int)tm[1]) * std::pow(q1, (int)tm[2]) * std::pow(q2, (int)tm[3]);
    }
    return s;
  }
};

template <class S>
void sh_analysis(const S& u, int N, int L, int qover, const double* centre, double* Fout) {
  const int R = N / 2, Lq = qover * L, nth = Lq + 1, nph = 2 * Lq + 2;
  vector<double> x, w;
  gauss_legendre(nth, x, w);
  vector<cd> tw((size_t)(L + 1) * nph);
  for (int m = 0; m <= L; ++m)
    for (int k = 0; k < nph; ++k) tw[(size_t)m * nph + k] = std::polar(1.0, -2.0 * PI * m * k / nph);
  vector<cd> F((size_t)ncoef(L) * R, cd(0, 0));
  vector<double> P, ring(nph);
  vector<cd> G(L + 1);
  for (int j = 0; j < nth; ++j) {
    const double ct = x[j], st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
    legendre_norm(L, ct, P);
    for (int i = 0; i < R; ++i) {
      const double r = i + 0.5;
      for (int k = 0; k < nph; ++k) {
        const double ph = 2.0 * PI * k / nph;
        ring[k] = u(centre[0] + r * st * std::cos(ph), centre[1] + r * st * std::sin(ph), centre[2] + r * ct);
      }
      for (int m = 0; m <= L; ++m) {
        cd s(0, 0);
        for (int k = 0; k < nph; ++k) s += ring[k] * tw[(size_t)m * nph + k];
        G[m] = s * (2.0 * PI / nph);
      }
      for (int l = 0; l <= L; ++l)
        for (int m = 0; m <= l; ++m) F[(size_t)lm_index(l, m) * R + i] += w[j] * P[lm_index(l, m)] * G[m];
    }
  }
  std::memcpy(Fout, F.data(), sizeof(cd) * F.size());
}

/* f_{l,-m} = (-1)^m conj(f_{lm}) for real u (reading C3) */
inline cd coef(const double* F, int R, int l, int m, int i) {
  const cd* c = reinterpret_cast<const cd*>(F);
  if (m >= 0) return c[(size_t)lm_index(l, m) * R + i];
  cd v = std::conj(c[(size_t)lm_index(l, -m) * R + i]);
  return (m % 2 == 0) ? v : -v;
}

/* ---------------- stage 2: Wigner coefficient tensor (north_star (2)) -----------
   M^l_{mn} = sum_i w_i f_lm(r_i) conj(h_ln(r_i)), w_i = r_i^2, all m,n in [-l,l] (full plane). */
void corr_full(const double* F, const double* H, int R, int Lc, double* Mout) {
  cd* M = reinterpret_cast<cd*>(Mout);
  for (int l = 0; l <= Lc; ++l)
    for (int m = -l; m <= l; ++m)
      for (int n = -l; n <= l; ++n) {
        cd s(0, 0);
        for (int i = 0; i < R; ++i) {
          double r = i + 0.5;
          s += r * r * coef(F, R, l, m, i) * std::conj(coef(H, R, l, n, i));
        }
        M[full_offset(l) + (m + l) * (2 * l + 1) + (n + l)] = s;
      }
}

/* ---------------- C_L and its derivatives (Eq. 4 P:114-122 with reading C1) ----
   C_L(g) = sum_{l<=L} sum_{m,n} conj(M^l_mn) D^l_mn(g),  D^l_mn = e^{-im a} d^l_mn(b) e^{-in g}
   out[0]=C, out[1..3]=grad (a,b,g), out[4..9]=hess (aa,bb,gg,ab,ag,bg). */
void eval_corr(const double* Mfull, int L, const double* e, double* out) {
  const cd* M = reinterpret_cast<const cd*>(Mfull);
  vector<vector<double>> d;
  wigner_d_all(L, e[1], d);
  double acc[10] = {0};
  vector<double> d1, d2;
  for (int l = 0; l <= L; ++l) {
    ladder(l, d[l], d1);
    ladder(l, d1, d2);
    const int w = 2 * l + 1;
    for (int m = -l; m <= l; ++m)
      for (int n = -l; n <= l; ++n) {
        const cd Mc = std::conj(M[full_offset(l) + (m + l) * w + (n + l)]);
        const cd ph = std::polar(1.0, -(m * e[0] + n * e[2]));
        const int id = (m + l) * w + (n + l);
        const cd D = ph * d[l][id], Db = ph * d1[id], Dbb = ph * d2[id];
        const cd im(0, -1.0 * m), in(0, -1.0 * n);
        acc[0] += std::real(Mc * D);
        acc[1] += std::real(Mc * im * D);
        acc[2] += std::real(Mc * Db);
        acc[3] += std::real(Mc * in * D);
        acc[4] += std::real(Mc * im * im * D);
        acc[5] += std::real(Mc * Dbb);
        acc[6] += std::real(Mc * in * in * D);
        acc[7] += std::real(Mc * im * Db);
        acc[8] += std::real(Mc * im * in * D);
        acc[9] += std::real(Mc * in * Db);
      }
  }
  for (int k = 0; k < 10; ++k) out[k] = acc[k];
}

/* ---------------- stage 3: coarse SO(3) grid (reading C9) ----------------
   grid[(j n_a + a) n_g + c] = C_{L0}(alpha_a, beta_j, gamma_c), evaluated DIRECTLY. */
void grid_dims(int L0, int K, int& nb, int& na, int& ng) {
  nb = K * (L0 + 1);
  na = ng = 2 * K * (L0 + 1);
}
/* worker threads a single particle's grid evaluation may use (set by orc_align_batch when particles are fewer
   than cores; the beta rows are independent, so the result does not depend on it) */
int g_inner_threads = 1;

template <class Fn> void parallel_for(int64_t n, int nthreads, Fn fn);

void grid_eval(const double* Mfull, int L0, int K, double* grid) {
  const cd* M = reinterpret_cast<const cd*>(Mfull);
  int nb, na, ng;
  grid_dims(L0, K, nb, na, ng);
  vector<cd> ea((size_t)(2 * L0 + 1) * na), eg((size_t)(2 * L0 + 1) * ng);
  for (int m = -L0; m <= L0; ++m)
    for (int a = 0; a < na; ++a) ea[(size_t)(m + L0) * na + a] = std::polar(1.0, -m * 2.0 * PI * a / na);
  for (int n = -L0; n <= L0; ++n)
    for (int c = 0; c < ng; ++c) eg[(size_t)(n + L0) * ng + c] = std::polar(1.0, -n * 2.0 * PI * c / ng);
  parallel_for(nb, g_inner_threads, [&](int64_t jj) {
    const int j = (int)jj;
    vector<vector<double>> d;
    const double beta = (j + 0.5) * PI / nb;
    wigner_d_all(L0, beta, d);
    for (int a = 0; a < na; ++a)
      for (int c = 0; c < ng; ++c) {
        double s = 0;
        for (int l = 0; l <= L0; ++l) {
          const int w = 2 * l + 1;
          for (int m = -l; m <= l; ++m)
            for (int n = -l; n <= l; ++n) {
              const cd D = ea[(size_t)(m + L0) * na + a] * d[l][(m + l) * w + (n + l)] * eg[(size_t)(n + L0) * ng + c];
              s += std::real(std::conj(M[full_offset(l) + (m + l) * w + (n + l)]) * D);
            }
        }
        grid[((size_t)j * na + a) * ng + c] = s;
      }
  });
}

/* local maxima ("N_C strongest local maxima"; readings C10, C11): node p is kept iff
   for each of its 26 neighbours q (alpha, gamma periodic, beta clamped):
   v_p > v_q or (v_p == v_q and idx_p < idx_q).  Ranked by (score desc, idx asc). */
int find_maxima(const double* grid, int nb, int na, int ng, int ncand, int64_t* idx_out, double* score_out) {
  struct Cand { double v; int64_t i; };
  vector<Cand> all;
  for (int j = 0; j < nb; ++j)
    for (int a = 0; a < na; ++a)
      for (int c = 0; c < ng; ++c) {
        const int64_t ip = ((int64_t)j * na + a) * ng + c;
        const double vp = grid[ip];
        bool is_max = true;
        for (int dj = -1; dj <= 1 && is_max; ++dj) {
          int jj = j + dj;
          if (jj < 0 || jj >= nb) continue;
          for (int da = -1; da <= 1 && is_max; ++da)
            for (int dc = -1; dc <= 1 && is_max; ++dc) {
              if (!dj && !da && !dc) continue;
              int aa = (a + da + na) % na, cc = (c + dc + ng) % ng;
              int64_t iq = ((int64_t)jj * na + aa) * ng + cc;
              if (iq == ip) continue;
              double vq = grid[iq];
              if (!(vp > vq || (vp == vq && ip < iq))) is_max = false;
            }
        }
        if (is_max) all.push_back({vp, ip});
      }
  std::sort(all.begin(), all.end(), [](const Cand& x, const Cand& y) {
    return x.v > y.v || (x.v == y.v && x.i < y.i);
  });
  int nfound = (int)std::min<size_t>(all.size(), (size_t)ncand);
  for (int k = 0; k < ncand; ++k) {
    if (k < nfound) {
      idx_out[k] = all[k].i;
      score_out[k] = all[k].v;
    } else {
      idx_out[k] = -1;
      score_out[k] = -std::numeric_limits<double>::infinity();
    }
  }
  return nfound;
}

void grid_node_euler(int64_t idx, int L0, int K, double* e) {
  int nb, na, ng;
  grid_dims(L0, K, nb, na, ng);
  int c = (int)(idx % ng);
  int a = (int)((idx / ng) % na);
  int j = (int)(idx / ((int64_t)ng * na));
  e[0] = 2.0 * PI * a / na;
  e[1] = (j + 0.5) * PI / nb;
  e[2] = 2.0 * PI * c / ng;
}

/* ---------------- stage 4: Newton step (readings C13, C15) ----------------
   H_reg = H if -H > 0, else H - (lambda_max(H) + 1e-6 ||H||_F) I;  delta = -H_reg^{-1} grad. */
void jacobi_eigenvalues(const double* Hs, double* ev) {
  double A[3][3] = {{Hs[0], Hs[3], Hs[4]}, {Hs[3], Hs[1], Hs[5]}, {Hs[4], Hs[5], Hs[2]}};
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
    double nrm = A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2] + 2 * off;
    if (off <= 1e-32 * nrm || off == 0.0) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (A[p][q] == 0.0) continue;
        double th = 0.5 * std::atan2(2 * A[p][q], A[q][q] - A[p][p]);
        double c = std::cos(th), s = std::sin(th);
        /* A <- J^T A J with J the (p,q) rotation */
        for (int k = 0; k < 3; ++k) {
          double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - s * akq;
          A[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - s * aqk;
          A[q][k] = s * apk + c * aqk;
        }
      }
  }
  ev[0] = A[0][0]; ev[1] = A[1][1]; ev[2] = A[2][2];
}

void newton_delta(const double* g, const double* h, double* delta) {
  /* h = (aa, bb, gg, ab, ag, bg) */
  double ev[3];
  jacobi_eigenvalues(h, ev);
  double lmax = std::max(ev[0], std::max(ev[1], ev[2]));
  double fro = std::sqrt(h[0] * h[0] + h[1] * h[1] + h[2] * h[2] + 2 * (h[3] * h[3] + h[4] * h[4] + h[5] * h[5]));
  double shift = (lmax < 0) ? 0.0 : (lmax + 1e-6 * fro);
  double A[3][4] = {{h[0] - shift, h[3], h[4], -g[0]},
                    {h[3], h[1] - shift, h[5], -g[1]},
                    {h[4], h[5], h[2] - shift, -g[2]}};
  /* Gaussian elimination with partial pivoting */
  for (int c = 0; c < 3; ++c) {
    int p = c;
    for (int r = c + 1; r < 3; ++r)
      if (std::fabs(A[r][c]) > std::fabs(A[p][c])) p = r;
    if (A[p][c] == 0.0) { delta[0] = delta[1] = delta[2] = 0.0; return; }
    if (p != c)
      for (int k = 0; k < 4; ++k) std::swap(A[p][k], A[c][k]);
    for (int r = c + 1; r < 3; ++r) {
      double f = A[r][c] / A[c][c];
      for (int k = c; k < 4; ++k) A[r][k] -= f * A[c][k];
    }
  }
  for (int r = 2; r >= 0; --r) {
    double s = A[r][3];
    for (int k = r + 1; k < 3; ++k) s -= A[r][k] * delta[k];
    delta[r] = s / A[r][r];
  }
}

/* Algorithm 1 lines 3-8 with readings C12 (Newton at every band, incl. L0),
   C14 (early stop), C23 (argmax, lowest n on ties).  euler [ncand][3] in/out. */
void refine(const double* Mfull, const int* bands, int nbands, int iters, int ncand, const int64_t* idx,
            double tol_grad, double tol_step, double tol_obj, double* euler, double* score, int* best) {
  for (int n = 0; n < ncand; ++n) {
    const bool active = !idx || idx[n] >= 0;
    if (!active) continue;
    double* th = euler + 3 * n;
    for (int j = 0; j < nbands; ++j) {
      double Cprev = 0;
      for (int s = 0; s < iters; ++s) {
        double out[10], delta[3];
        eval_corr(Mfull, bands[j], th, out);
        double gn = std::sqrt(out[1] * out[1] + out[2] * out[2] + out[3] * out[3]);
        if (tol_grad > 0 && gn < tol_grad * std::fabs(out[0])) break;
        if (s > 0 && tol_obj > 0 && std::fabs(out[0] - Cprev) < tol_obj * std::fabs(out[0])) break;
        newton_delta(out + 1, out + 4, delta);
        for (int k = 0; k < 3; ++k) th[k] += delta[k];
        canon(th);
        Cprev = out[0];
        double dn = std::sqrt(delta[0] * delta[0] + delta[1] * delta[1] + delta[2] * delta[2]);
        if (tol_step > 0 && dn < tol_step) break;
      }
    }
  }
  const int LJ = bands[nbands - 1];
  int b = -1;
  for (int n = 0; n < ncand; ++n) {
    const bool active = !idx || idx[n] >= 0;
    if (!active) { score[n] = -std::numeric_limits<double>::infinity(); continue; }
    double out[10];
    eval_corr(Mfull, LJ, euler + 3 * n, out);
    score[n] = out[0];
    if (b < 0 || score[n] > score[b]) b = n;
  }
  *best = b;
}

/* ---------------- stage 5: translation (App. C; readings C17, C18) ----------------
   rho(x) = h(R^T (x - c) + c) (trilinear, zero outside);  c(t) = sum_x f(x) rho((x - t) mod N),
   argmax over t in [-W,W]^3 (tie -> lowest window index, z-major), parabolic subpixel per axis. */
void rotate_volume(const float* ref, int N, const double* e, vector<double>& out) {
  double R[9];
  euler_to_matrix(e, R);
  VolSampler s{ref, N};
  const double c = 0.5 * (N - 1);
  out.assign((size_t)N * N * N, 0.0);
  for (int z = 0; z < N; ++z)
    for (int y = 0; y < N; ++y)
      for (int x = 0; x < N; ++x) {
        double v0 = x - c, v1 = y - c, v2 = z - c;
        double q0 = R[0] * v0 + R[3] * v1 + R[6] * v2;
        double q1 = R[1] * v0 + R[4] * v1 + R[7] * v2;
        double q2 = R[2] * v0 + R[5] * v1 + R[8] * v2;
        out[((size_t)z * N + y) * N + x] = s(q0 + c, q1 + c, q2 + c);
      }
}

double circ_corr(const float* f, const vector<double>& rho, int N, int tx, int ty, int tz) {
  double s = 0;
  for (int z = 0; z < N; ++z) {
    int zz = ((z - tz) % N + N) % N;
    for (int y = 0; y < N; ++y) {
      int yy = ((y - ty) % N + N) % N;
      const float* fr = f + ((size_t)z * N + y) * N;
      const double* rr = rho.data() + ((size_t)zz * N + yy) * N;
      for (int x = 0; x < N; ++x) {
        int xx = ((x - tx) % N + N) % N;
        s += (double)fr[x] * rr[xx];
      }
    }
  }
  return s;
}

void translation(const float* vol, const float* ref, int N, const double* e, int W, double* shift, double* peak) {
  vector<double> rho;
  rotate_volume(ref, N, e, rho);
  double best = -std::numeric_limits<double>::infinity();
  int bt[3] = {0, 0, 0};
  for (int tz = -W; tz <= W; ++tz)
    for (int ty = -W; ty <= W; ++ty)
      for (int tx = -W; tx <= W; ++tx) {
        double v = circ_corr(vol, rho, N, tx, ty, tz);
        if (v > best) { best = v; bt[0] = tx; bt[1] = ty; bt[2] = tz; } /* scan order = window index order */
      }
  *peak = best;
  for (int ax = 0; ax < 3; ++ax) {
    int tm[3] = {bt[0], bt[1], bt[2]}, tp[3] = {bt[0], bt[1], bt[2]};
    tm[ax] -= 1;
    tp[ax] += 1;
    double cm = circ_corr(vol, rho, N, tm[0], tm[1], tm[2]);
    double cp = circ_corr(vol, rho, N, tp[0], tp[1], tp[2]);
    double den = cm - 2 * best + cp;
    double dlt = 0;
    if (den < 0) dlt = std::max(-0.5, std::min(0.5, (cm - cp) / (2 * den)));
    shift[ax] = bt[ax] + dlt;
  }
}

/* ---------------- stage 5, subpixel by an upsampled DFT (App. C remark iii) ----------------
   Guizar-Sicairos's scheme: the integer peak t0 of the windowed correlation (as translation() above), then the
   correlation's trigonometric interpolant on a kappa-times finer grid over +-1.5 voxel around t0, evaluated by
   matrix-multiply DFTs (reading C27: the REAL trigonometric interpolant, the Nyquist index N/2 split evenly
   between +-N/2, i.e. D(N/2, t) = cos(pi t)):
     c~(t) = (1/N^3) sum_{k in [0,N)^3} F^(k) conj(rho^(k)) D(kx, tx) D(ky, ty) D(kz, tz),
     D(k, t) = e^{+2 pi i k' t / N} with k' = k (k < N/2) or k - N (k > N/2), D(N/2, t) = cos(pi t),
   F^, rho^ the 3-D DFTs of f and rho (here by a plain separable DFT in FP64), t = t0 + u / kappa,
   u in [-h, h]^3 with h = ceil(1.5 kappa); the result is the argmax (ties -> lowest index, z-major) and c~ there.
   At integer t, c~(t) = c(t) = sum_x f(x) rho(x - t) exactly (circular correlation). */
void dft_axis(vector<cd>& a, int N, int axis) {
  /* a: [z][y][x] complex N^3; forward DFT e^{-2 pi i k n / N} along one axis, by the definition */
  vector<cd> w(N);
  for (int m = 0; m < N; ++m) w[m] = std::polar(1.0, -2.0 * PI * m / N);
  vector<cd> line(N), out(N);
  const size_t st = axis == 0 ? 1 : axis == 1 ? (size_t)N : (size_t)N * N;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      size_t base;
      if (axis == 0) base = ((size_t)i * N + j) * N;
      else if (axis == 1) base = (size_t)i * N * N + j;
      else base = (size_t)i * N + j;
      for (int n = 0; n < N; ++n) line[n] = a[base + n * st];
      for (int k = 0; k < N; ++k) {
        cd s(0, 0);
        for (int n = 0; n < N; ++n) s += line[n] * w[((size_t)k * n) % N];
        out[k] = s;
      }
      for (int k = 0; k < N; ++k) a[base + k * st] = out[k];
    }
}

cd interp_kernel(int k, int N, double t) {
  if (2 * k == N) return cd(std::cos(PI * t), 0.0);
  const int kp = k < N / 2 ? k : k - N;
  return std::polar(1.0, 2.0 * PI * kp * t / N);
}

void translation_upsampled(const float* vol, const float* ref, int N, const double* e, int W, int kappa,
                           double* shift, double* peak) {
  double tpar[3], pk;
  translation(vol, ref, N, e, W, tpar, &pk);  /* parabolic result; its integer part is recomputed below */
  vector<double> rho;
  rotate_volume(ref, N, e, rho);
  /* integer window argmax t0 (same scan as translation) */
  double best = -std::numeric_limits<double>::infinity();
  int t0[3] = {0, 0, 0};
  for (int tz = -W; tz <= W; ++tz)
    for (int ty = -W; ty <= W; ++ty)
      for (int tx = -W; tx <= W; ++tx) {
        double v = circ_corr(vol, rho, N, tx, ty, tz);
        if (v > best) { best = v; t0[0] = tx; t0[1] = ty; t0[2] = tz; }
      }
  const size_t n3 = (size_t)N * N * N;
  vector<cd> F(n3), R(n3);
  for (size_t i = 0; i < n3; ++i) { F[i] = cd(vol[i], 0.0); R[i] = cd(rho[i], 0.0); }
  for (int ax = 0; ax < 3; ++ax) { dft_axis(F, N, ax); dft_axis(R, N, ax); }
  vector<cd> X(n3);
  for (size_t i = 0; i < n3; ++i) X[i] = F[i] * std::conj(R[i]);
  const int h = (int)std::ceil(1.5 * kappa), U = 2 * h + 1;
  /* phase matrices E_ax[k][u] = D(k, t0_ax + (u - h)/kappa) */
  vector<cd> E[3];
  for (int ax = 0; ax < 3; ++ax) {
    E[ax].resize((size_t)N * U);
    for (int k = 0; k < N; ++k)
      for (int u = 0; u < U; ++u) E[ax][(size_t)k * U + u] = interp_kernel(k, N, t0[ax] + (double)(u - h) / kappa);
  }
  /* separable contraction: x, then y, then z (matrix-multiply DFTs) */
  vector<cd> A((size_t)N * N * U), B((size_t)N * U * U);
  for (int z = 0; z < N; ++z)
    for (int y = 0; y < N; ++y)
      for (int u = 0; u < U; ++u) {
        cd s(0, 0);
        for (int kx = 0; kx < N; ++kx) s += X[((size_t)z * N + y) * N + kx] * E[0][(size_t)kx * U + u];
        A[((size_t)z * N + y) * U + u] = s;
      }
  for (int z = 0; z < N; ++z)
    for (int v = 0; v < U; ++v)
      for (int u = 0; u < U; ++u) {
        cd s(0, 0);
        for (int ky = 0; ky < N; ++ky) s += A[((size_t)z * N + ky) * U + u] * E[1][(size_t)ky * U + v];
        B[((size_t)z * U + v) * U + u] = s;
      }
  double bv = -std::numeric_limits<double>::infinity();
  int bu[3] = {h, h, h};
  for (int w = 0; w < U; ++w)
    for (int v = 0; v < U; ++v)
      for (int u = 0; u < U; ++u) {
        cd s(0, 0);
        for (int kz = 0; kz < N; ++kz) s += B[((size_t)kz * U + v) * U + u] * E[2][(size_t)kz * U + w];
        const double c = std::real(s) / (double)n3;  /* imaginary part 0 up to rounding (Hermitian X, real D) */
        if (c > bv) { bv = c; bu[0] = u; bu[1] = v; bu[2] = w; } /* scan order = z-major index order */
      }
  for (int ax = 0; ax < 3; ++ax) shift[ax] = t0[ax] + (double)(bu[ax] - h) / kappa;
  *peak = bv;
}

/* ---------------- ball-harmonic radial basis (App. A.1; reading C30) ----------------
   j_l(x) = (1/2) (-i)^l int_{-1}^{1} e^{i x t} P_l(t) dt (the plane-wave integral, by Gauss-Legendre quadrature
   with n_q >= x/2 + l + 40 nodes: exact to rounding for this entire integrand); lambda_lk the k-th positive root of
   j_l (sign changes on a 0.05 grid, then bisection); c_lk = sqrt(2)/|j_{l+1}(lambda_lk)|;
   f^_klm = sum_i (1/R) rho_i^2 c_lk j_l(lambda_lk rho_i) f_lm(r_i), rho_i = (i - 1/2)/R;
   M^l_mn = sum_{k in K_l} f^_klm conj(h^_kln). */
struct SphBessel {
  int L, nq;
  vector<double> t, w, P;  /* nodes, weights, P[l * nq + q] = P_l(t_q) */
  SphBessel(int L_, double xmax) : L(L_) {
    nq = (int)(xmax / 2 + L + 40);
    gauss_legendre(nq, t, w);
    P.assign((size_t)(L + 2) * nq, 0.0);
    for (int q = 0; q < nq; ++q) {
      double p0 = 1.0, p1 = t[q];
      P[q] = 1.0;
      if (L + 1 >= 1) P[nq + q] = p1;
      for (int l = 2; l <= L + 1; ++l) {
        const double p2 = ((2.0 * l - 1.0) * t[q] * p1 - (l - 1.0) * p0) / l;
        P[(size_t)l * nq + q] = p2;
        p0 = p1;
        p1 = p2;
      }
    }
  }
  double operator()(int l, double x) const {
    cd s(0, 0);
    for (int q = 0; q < nq; ++q) s += w[q] * P[(size_t)l * nq + q] * std::polar(1.0, x * t[q]);
    cd f(1, 0);
    for (int k = 0; k < l % 4; ++k) f *= cd(0, -1);
    return 0.5 * std::real(f * s);
  }
};

void ball_tables(int L, int R, double lam, vector<int>& K, vector<vector<double>>& Bt) {
  if (lam <= 0) lam = PI * (R - 0.5);
  SphBessel jl(L, lam + 1.0);
  K.assign(L + 1, 0);
  Bt.assign(L + 1, vector<double>());
  for (int l = 0; l <= L; ++l) {
    vector<double> roots;
    double x0 = std::max(0.5, (double)l), f0 = jl(l, x0);
    for (double x1 = x0 + 0.05; x0 <= lam; x1 += 0.05) {
      const double f1 = jl(l, x1);
      if (f0 == 0.0 || f0 * f1 < 0.0) {
        double a = x0, b = x1, fa = f0;
        for (int it = 0; it < 200 && b - a > 1e-15 * b; ++it) {
          const double m = 0.5 * (a + b), fm = jl(l, m);
          if ((fm < 0) == (fa < 0)) { a = m; fa = fm; } else { b = m; }
        }
        if (0.5 * (a + b) <= lam) roots.push_back(0.5 * (a + b));
      }
      x0 = x1;
      f0 = f1;
    }
    if ((int)roots.size() > R) roots.resize(R);
    K[l] = (int)roots.size();
    Bt[l].assign((size_t)K[l] * R, 0.0);
    for (int k = 0; k < K[l]; ++k) {
      const double c = std::sqrt(2.0) / std::fabs(jl(l + 1, roots[k]));
      for (int i = 0; i < R; ++i) {
        const double rho = (i + 0.5) / R;
        Bt[l][(size_t)k * R + i] = rho * rho / R * c * jl(l, roots[k] * rho);
      }
    }
  }
}

/* F complex [ncoef(L)][R] -> Fb complex [ncoef(L)][Kmax] */
void ball_transform(const double* F, int L, int R, const vector<int>& K, const vector<vector<double>>& Bt, int Kmax,
                    double* Fb) {
  const cd* f = reinterpret_cast<const cd*>(F);
  cd* o = reinterpret_cast<cd*>(Fb);
  for (int l = 0; l <= L; ++l)
    for (int m = 0; m <= l; ++m)
      for (int k = 0; k < Kmax; ++k) {
        cd s(0, 0);
        if (k < K[l])
          for (int i = 0; i < R; ++i) s += Bt[l][(size_t)k * R + i] * f[(size_t)lm_index(l, m) * R + i];
        o[(size_t)lm_index(l, m) * Kmax + k] = s;
      }
}

/* full-plane M^l_mn = sum_{k < K_l} f^_klm conj(h^_kln), all m, n (reality of f, h: reading C3) */
void corr_ball_full(const double* Fb, const double* Hb, const vector<int>& K, int Kmax, int Lc, double* Mout) {
  cd* M = reinterpret_cast<cd*>(Mout);
  for (int l = 0; l <= Lc; ++l)
    for (int m = -l; m <= l; ++m)
      for (int n = -l; n <= l; ++n) {
        cd s(0, 0);
        for (int k = 0; k < K[l]; ++k) s += coef(Fb, Kmax, l, m, k) * std::conj(coef(Hb, Kmax, l, n, k));
        M[full_offset(l) + (m + l) * (2 * l + 1) + (n + l)] = s;
      }
}

struct Params {
  int L, qover, L0, K, ncand, nbands, bands[16], iters, T, W, ups, radial;
  double tol_grad, tol_step, tol_obj, lambda;
};

/* whole path for one particle: App. C alternation around Algorithm 1 (reading C19). */
void align_one(const float* vol, const float* ref, const double* H, int N, const Params& p, double* pose) {
  const int R = N / 2;
  const double c = 0.5 * (N - 1);
  double t[3] = {0, 0, 0};
  vector<double> F((size_t)2 * ncoef(p.L) * R), M((size_t)2 * full_size(p.L));
  int nb, na, ng;
  grid_dims(p.L0, p.K, nb, na, ng);
  vector<double> grid((size_t)nb * na * ng);
  vector<int64_t> idx(p.ncand);
  vector<double> sc(p.ncand), eu((size_t)3 * p.ncand);
  int best = -1;
  double rot[3] = {0, 0, 0}, score = 0;
  for (int tau = 0; tau < std::max(1, p.T); ++tau) {
    double centre[3] = {c + t[0], c + t[1], c + t[2]};
    sh_analysis(VolSampler{vol, N}, N, p.L, p.qover, centre, F.data());
    if (p.radial == 1) {
      /* M from the ball-harmonic coefficients (tables per call: plain, slow) */
      vector<int> K;
      vector<vector<double>> Bt;
      ball_tables(p.L, R, p.lambda, K, Bt);
      int Kmax = 0;
      for (int k : K) Kmax = std::max(Kmax, k);
      vector<double> Fb((size_t)2 * ncoef(p.L) * Kmax), Hb((size_t)2 * ncoef(p.L) * Kmax);
      ball_transform(F.data(), p.L, R, K, Bt, Kmax, Fb.data());
      ball_transform(H, p.L, R, K, Bt, Kmax, Hb.data());
      corr_ball_full(Fb.data(), Hb.data(), K, Kmax, p.L, M.data());
    } else {
      corr_full(F.data(), H, R, p.L, M.data());
    }
    grid_eval(M.data(), p.L0, p.K, grid.data());
    find_maxima(grid.data(), nb, na, ng, p.ncand, idx.data(), sc.data());
    for (int n = 0; n < p.ncand; ++n) {
      if (idx[n] >= 0) grid_node_euler(idx[n], p.L0, p.K, &eu[3 * n]);
      else eu[3 * n] = eu[3 * n + 1] = eu[3 * n + 2] = 0.0;
    }
    refine(M.data(), p.bands, p.nbands, p.iters, p.ncand, idx.data(), p.tol_grad, p.tol_step, p.tol_obj, eu.data(),
           sc.data(), &best);
    if (best >= 0) {
      for (int k = 0; k < 3; ++k) rot[k] = eu[3 * best + k];
      score = sc[best];
    }
    if (p.W > 0) {
      double pk;
      if (p.ups > 0) translation_upsampled(vol, ref, N, rot, p.W, p.ups, t, &pk);
      else translation(vol, ref, N, rot, p.W, t, &pk);
    }
  }
  pose[0] = rot[0]; pose[1] = rot[1]; pose[2] = rot[2];
  pose[3] = t[0]; pose[4] = t[1]; pose[5] = t[2];
  pose[6] = score; pose[7] = best;
}

/* ||H_{<=L}||_w = sqrt(sum_i w_i sum_{l<=L} sum_{m=-l..l} |h_lm(r_i)|^2): the template's band-limited norm (the
   Cauchy-Schwarz scale of C_L, SURVEY 8(c) tolerances) */
double template_norm(const double* H, int L, int R) {
  double e = 0;
  for (int l = 0; l <= L; ++l)
    for (int m = -l; m <= l; ++m)
      for (int i = 0; i < R; ++i) {
        const double r = i + 0.5;
        e += r * r * std::norm(coef(H, R, l, m, i));
      }
  return std::sqrt(e);
}

/* whole path for one particle against nt templates: per alternation the rotation search of
   align_one against every template; the template with the highest C_{L_J} / ||H_{<=L_J}||_w wins (reading C29: the
   raw inner product grows with the template's energy, the particle's norm is common to all templates; ties -> the
   lowest template index); the translation update rotates the winning template.
   pose [9] = {alpha, beta, gamma, tx, ty, tz, score (raw C_{L_J}), best, template}. */
void align_one_multi(const float* vol, const float* refs, int nt, const double* Hs, int N, const Params& p,
                     double* pose) {
  const int R = N / 2;
  const size_t n3 = (size_t)N * N * N, hsz = (size_t)2 * ncoef(p.L) * R;
  const double c = 0.5 * (N - 1);
  double t[3] = {0, 0, 0};
  vector<double> F(hsz), M((size_t)2 * full_size(p.L));
  int nb, na, ng;
  grid_dims(p.L0, p.K, nb, na, ng);
  vector<double> grid((size_t)nb * na * ng);
  vector<int64_t> idx(p.ncand);
  vector<double> sc(p.ncand), eu((size_t)3 * p.ncand);
  double rot[3] = {0, 0, 0}, score = 0, nbest = 0;
  int best = -1, tbest = 0;
  for (int tau = 0; tau < std::max(1, p.T); ++tau) {
    double centre[3] = {c + t[0], c + t[1], c + t[2]};
    sh_analysis(VolSampler{vol, N}, N, p.L, p.qover, centre, F.data());
    bool have = false;
    for (int k = 0; k < nt; ++k) {
      corr_full(F.data(), Hs + k * hsz, R, p.L, M.data());
      grid_eval(M.data(), p.L0, p.K, grid.data());
      find_maxima(grid.data(), nb, na, ng, p.ncand, idx.data(), sc.data());
      for (int n = 0; n < p.ncand; ++n) {
        if (idx[n] >= 0) grid_node_euler(idx[n], p.L0, p.K, &eu[3 * n]);
        else eu[3 * n] = eu[3 * n + 1] = eu[3 * n + 2] = 0.0;
      }
      int b = -1;
      refine(M.data(), p.bands, p.nbands, p.iters, p.ncand, idx.data(), p.tol_grad, p.tol_step, p.tol_obj, eu.data(),
             sc.data(), &b);
      const double nk = sc[b >= 0 ? b : 0] / template_norm(Hs + k * hsz, p.bands[p.nbands - 1], R);
      if (b >= 0 && (!have || nk > nbest)) {
        have = true;
        nbest = nk;
        score = sc[b];
        best = b;
        tbest = k;
        for (int q = 0; q < 3; ++q) rot[q] = eu[3 * b + q];
      }
    }
    if (p.W > 0) {
      double pk;
      if (p.ups > 0) translation_upsampled(vol, refs + tbest * n3, N, rot, p.W, p.ups, t, &pk);
      else translation(vol, refs + tbest * n3, N, rot, p.W, t, &pk);
    }
  }
  pose[0] = rot[0]; pose[1] = rot[1]; pose[2] = rot[2];
  pose[3] = t[0]; pose[4] = t[1]; pose[5] = t[2];
  pose[6] = score; pose[7] = best; pose[8] = tbest;
}

/* reference update (P:1184 half sets; reading C28): sums[k][s][y] = sum over particles p of class k and
   half s = (first + p) mod 2 of f_p(g_p (y - c) + c + t_p) (trilinear, zero outside), counts[k][s]. */
void reconstruct(const float* vols, int64_t B, int N, const double* poses, int stride, int ccol, int ncls,
                 int64_t first, double* sums, int* counts) {
  const size_t n3 = (size_t)N * N * N;
  const double c = 0.5 * (N - 1);
  std::fill(sums, sums + (size_t)ncls * 2 * n3, 0.0);
  std::fill(counts, counts + 2 * ncls, 0);
  for (int64_t p = 0; p < B; ++p) {
    const double* ps = poses + p * stride;
    const int k = ccol >= 0 ? (int)ps[ccol] : 0;
    if (k < 0 || k >= ncls) continue;
    const int half = (int)((first + p) % 2);
    counts[2 * k + half] += 1;
    double Rm[9];
    euler_to_matrix(ps, Rm);
    VolSampler f{vols + p * n3, N};
    double* out = sums + (size_t)(2 * k + half) * n3;
    for (int z = 0; z < N; ++z)
      for (int y = 0; y < N; ++y)
        for (int x = 0; x < N; ++x) {
          const double u0 = x - c, u1 = y - c, u2 = z - c;
          const double q0 = Rm[0] * u0 + Rm[1] * u1 + Rm[2] * u2 + c + ps[3];
          const double q1 = Rm[3] * u0 + Rm[4] * u1 + Rm[5] * u2 + c + ps[4];
          const double q2 = Rm[6] * u0 + Rm[7] * u1 + Rm[8] * u2 + c + ps[5];
          out[((size_t)z * N + y) * N + x] += f(q0, q1, q2);
        }
  }
}

template <class Fn>
void parallel_for(int64_t n, int nthreads, Fn fn) {
  if (nthreads == 1 || n <= 1) {
    for (int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  nthreads = (int)std::min<int64_t>(nthreads, std::max<int64_t>(1, n));
  std::atomic<int64_t> next(0);
  vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back([&]() {
      for (;;) {
        int64_t i = next.fetch_add(1);
        if (i >= n) break;
        fn(i);
      }
    });
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

void orc_euler_to_matrix(const double* e, double* R) { euler_to_matrix(e, R); }
void orc_matrix_to_euler(const double* R, double* e) { matrix_to_euler(R, e); }
void orc_canon(double* e) { canon(e); }
void orc_gauss_legendre(int n, double* x, double* w) {
  vector<double> xv, wv;
  gauss_legendre(n, xv, wv);
  std::memcpy(x, xv.data(), sizeof(double) * n);
  std::memcpy(w, wv.data(), sizeof(double) * n);
}
void orc_legendre_norm(int L, double x, double* P) {
  vector<double> v;
  legendre_norm(L, x, v);
  std::memcpy(P, v.data(), sizeof(double) * v.size());
}
/* d, d1, d2: (2l+1)^2 row-major, m (row) and n (column) from -l..l; d1/d2 may be NULL */
void orc_wigner_d(int l, double beta, double* d, double* d1, double* d2) {
  vector<vector<double>> all;
  wigner_d_all(l, beta, all);
  std::memcpy(d, all[l].data(), sizeof(double) * all[l].size());
  vector<double> a, b;
  if (d1 || d2) ladder(l, all[l], a);
  if (d1) std::memcpy(d1, a.data(), sizeof(double) * a.size());
  if (d2) {
    ladder(l, a, b);
    std::memcpy(d2, b.data(), sizeof(double) * b.size());
  }
}
void orc_sh_analysis_vol(const float* vol, int N, int L, int qover, const double* shift, double* F) {
  const double c = 0.5 * (N - 1);
  double centre[3] = {c, c, c};
  if (shift)
    for (int k = 0; k < 3; ++k) centre[k] += shift[k];
  sh_analysis(VolSampler{vol, N}, N, L, qover, centre, F);
}
void orc_sh_analysis_poly(const double* terms, int nterms, const double* R9, int N, int L, int qover, double* F) {
  const double c = 0.5 * (N - 1);
  PolySampler s{terms, nterms, {1, 0, 0, 0, 1, 0, 0, 0, 1}, c, c, c};
  if (R9) std::memcpy(s.R, R9, sizeof(s.R));
  double centre[3] = {c, c, c};
  sh_analysis(s, N, L, qover, centre, F);
}
void orc_sh_analysis_batch(const float* vols, int64_t B, int N, int L, int qover, const double* shifts, double* F,
                           int nthreads) {
  const int R = N / 2;
  const size_t n3 = (size_t)N * N * N, fs = (size_t)2 * ncoef(L) * R;
  parallel_for(B, nthreads, [&](int64_t b) {
    orc_sh_analysis_vol(vols + b * n3, N, L, qover, shifts ? shifts + 3 * b : nullptr, F + b * fs);
  });
}
long orc_full_size(int L) { return full_size(L); }
/* F, H: complex [ncoef(L)][R] (L >= Lc); M: complex full-plane blocks l <= Lc */
void orc_corr_full(const double* F, const double* H, int L, int Lc, int R, double* M) {
  (void)L;
  corr_full(F, H, R, Lc, M);
}
void orc_eval_corr(const double* M, int L, const double* e, double* out10) { eval_corr(M, L, e, out10); }
void orc_grid_eval(const double* M, int L0, int K, double* grid) {
  g_inner_threads = (int)std::max(1u, std::thread::hardware_concurrency());  /* rows are independent */
  grid_eval(M, L0, K, grid);
  g_inner_threads = 1;
}
int orc_find_maxima(const double* grid, int nb, int na, int ng, int ncand, int64_t* idx, double* score) {
  return find_maxima(grid, nb, na, ng, ncand, idx, score);
}
void orc_grid_node_euler(int64_t idx, int L0, int K, double* e) { grid_node_euler(idx, L0, K, e); }
void orc_newton_delta(const double* g, const double* h, double* delta) { newton_delta(g, h, delta); }
void orc_refine(const double* M, const int* bands, int nbands, int iters, int ncand, const int64_t* idx,
                double tol_grad, double tol_step, double tol_obj, double* euler, double* score, int* best) {
  refine(M, bands, nbands, iters, ncand, idx, tol_grad, tol_step, tol_obj, euler, score, best);
}
void orc_rotate_volume(const float* ref, int N, const double* e, double* out) {
  vector<double> v;
  rotate_volume(ref, N, e, v);
  std::memcpy(out, v.data(), sizeof(double) * v.size());
}
void orc_translation(const float* vol, const float* ref, int N, const double* e, int W, double* shift, double* peak) {
  translation(vol, ref, N, e, W, shift, peak);
}
void orc_translation_upsampled(const float* vol, const float* ref, int N, const double* e, int W, int kappa,
                               double* shift, double* peak) {
  translation_upsampled(vol, ref, N, e, W, kappa, shift, peak);
}
/* c~(t) of the upsampled scheme at ONE arbitrary point t, by the full triple sum over k in K^3 (no separation):
   the pin of the separable contraction above */
double orc_upsampled_corr_at(const float* vol, const float* ref, int N, const double* e, const double* t) {
  vector<double> rho;
  rotate_volume(ref, N, e, rho);
  const size_t n3 = (size_t)N * N * N;
  vector<cd> F(n3), R(n3);
  for (size_t i = 0; i < n3; ++i) { F[i] = cd(vol[i], 0.0); R[i] = cd(rho[i], 0.0); }
  for (int ax = 0; ax < 3; ++ax) { dft_axis(F, N, ax); dft_axis(R, N, ax); }
  cd s(0, 0);
  for (int kz = 0; kz < N; ++kz)
    for (int ky = 0; ky < N; ++ky)
      for (int kx = 0; kx < N; ++kx) {
        const size_t i = ((size_t)kz * N + ky) * N + kx;
        s += F[i] * std::conj(R[i]) * interp_kernel(kx, N, t[0]) * interp_kernel(ky, N, t[1]) * interp_kernel(kz, N, t[2]);
      }
  return std::real(s) / (double)n3;
}
/* E_L = ||F_{<=L}||_w ||H_{<=L}||_w (SURVEY 8(c) tolerance scale; Cauchy-Schwarz bound on |C_L|) */
double orc_energy(const double* F, const double* H, int Lc, int R) {
  double ef = 0, eh = 0;
  for (int l = 0; l <= Lc; ++l)
    for (int m = -l; m <= l; ++m)
      for (int i = 0; i < R; ++i) {
        double r = i + 0.5;
        ef += r * r * std::norm(coef(F, R, l, m, i));
        eh += r * r * std::norm(coef(H, R, l, m, i));
      }
  return std::sqrt(ef * eh);
}
/* params: ints [L, qover, L0, K, ncand, nbands, bands[16], iters, T, W, ups, radial];
   dbl [tol_grad, tol_step, tol_obj, lambda]  (ups = 0: parabolic subpixel; ups = kappa > 0: the upsampled DFT of
   translation_upsampled; radial = 1: the ball-harmonic basis with cutoff lambda)
   H: complex [ncoef(L)][R] reference coefficients (NULL -> analysed from ref at t = 0).
   poses [B][8] = {alpha, beta, gamma, tx, ty, tz, score, best}. */
void orc_align_batch(const float* vols, int64_t B, const float* ref, const double* H, int N, const int* ip,
                     const double* dp, double* poses, int nthreads) {
  Params p;
  p.L = ip[0]; p.qover = ip[1]; p.L0 = ip[2]; p.K = ip[3]; p.ncand = ip[4]; p.nbands = ip[5];
  for (int k = 0; k < 16; ++k) p.bands[k] = ip[6 + k];
  p.iters = ip[22]; p.T = ip[23]; p.W = ip[24]; p.ups = ip[25]; p.radial = ip[26];
  p.tol_grad = dp[0]; p.tol_step = dp[1]; p.tol_obj = dp[2]; p.lambda = dp[3];
  const int R = N / 2;
  vector<double> Hl;
  if (!H) {
    Hl.resize((size_t)2 * ncoef(p.L) * R);
    orc_sh_analysis_vol(ref, N, p.L, p.qover, nullptr, Hl.data());
    H = Hl.data();
  }
  const size_t n3 = (size_t)N * N * N;
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  const int outer = nthreads > 0 ? nthreads : hw;
  g_inner_threads = (int)std::max<int64_t>(1, outer / std::max<int64_t>(1, std::min<int64_t>(B, outer)));
  parallel_for(B, nthreads, [&](int64_t b) { align_one(vols + b * n3, ref, H, N, p, poses + 8 * b); });
  g_inner_threads = 1;
}

/* multi-template: refs float [nt][N^3]; Hs complex [nt][ncoef(L)][R] or NULL (analysed here); poses [B][9] */
void orc_align_batch_multi(const float* vols, int64_t B, const float* refs, int nt, const double* Hs, int N,
                           const int* ip, const double* dp, double* poses, int nthreads) {
  Params p;
  p.L = ip[0]; p.qover = ip[1]; p.L0 = ip[2]; p.K = ip[3]; p.ncand = ip[4]; p.nbands = ip[5];
  for (int k = 0; k < 16; ++k) p.bands[k] = ip[6 + k];
  p.iters = ip[22]; p.T = ip[23]; p.W = ip[24]; p.ups = ip[25]; p.radial = 0;
  p.tol_grad = dp[0]; p.tol_step = dp[1]; p.tol_obj = dp[2]; p.lambda = 0;
  const int R = N / 2;
  const size_t n3 = (size_t)N * N * N, hsz = (size_t)2 * ncoef(p.L) * R;
  vector<double> Hl;
  if (!Hs) {
    Hl.resize(hsz * nt);
    for (int k = 0; k < nt; ++k) orc_sh_analysis_vol(refs + k * n3, N, p.L, p.qover, nullptr, Hl.data() + k * hsz);
    Hs = Hl.data();
  }
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  const int outer = nthreads > 0 ? nthreads : hw;
  g_inner_threads = (int)std::max<int64_t>(1, outer / std::max<int64_t>(1, std::min<int64_t>(B, outer)));
  parallel_for(B, nthreads, [&](int64_t b) { align_one_multi(vols + b * n3, refs, nt, Hs, N, p, poses + 9 * b); });
  g_inner_threads = 1;
}
void orc_reconstruct(const float* vols, int64_t B, int N, const double* poses, int stride, int ccol, int ncls,
                     int64_t first, double* sums, int* counts) {
  reconstruct(vols, B, N, poses, stride, ccol, ncls, first, sums, counts);
}

/* ball basis: K [L+1] (|K_l|), returns Kmax; Bt [L+1][Kmax][R] if not NULL */
int orc_ball_tables(int L, int R, double lambda, int* K, double* Bt) {
  vector<int> Kv;
  vector<vector<double>> Bv;
  ball_tables(L, R, lambda, Kv, Bv);
  int Kmax = 0;
  for (int k : Kv) Kmax = std::max(Kmax, k);
  for (int l = 0; l <= L; ++l) {
    K[l] = Kv[l];
    if (Bt)
      for (int k = 0; k < Kmax; ++k)
        for (int i = 0; i < R; ++i) Bt[((size_t)l * Kmax + k) * R + i] = k < Kv[l] ? Bv[l][(size_t)k * R + i] : 0.0;
  }
  return Kmax;
}
double orc_sph_bessel(int l, double x) { return SphBessel(l, x + 1.0)(l, x); }
void orc_ball_transform(const double* F, int L, int R, double lambda, double* Fb) {
  vector<int> K;
  vector<vector<double>> Bt;
  ball_tables(L, R, lambda, K, Bt);
  int Kmax = 0;
  for (int k : K) Kmax = std::max(Kmax, k);
  ball_transform(F, L, R, K, Bt, Kmax, Fb);
}
void orc_corr_ball_full(const double* Fb, const double* Hb, int L, int R, double lambda, int Lc, double* M) {
  vector<int> K;
  vector<vector<double>> Bt;
  ball_tables(L, R, lambda, K, Bt);
  int Kmax = 0;
  for (int k : K) Kmax = std::max(Kmax, k);
  corr_ball_full(Fb, Hb, K, Kmax, Lc, M);
}

}  // extern "C"
