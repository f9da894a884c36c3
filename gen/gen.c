/*
 * gen.c -- seeded synthetic-input generator shared by the oracle tests and the GPU path.
 *
 * This module holds NONE of the method's arithmetic (no spherical harmonics, no Wigner
 * functions, no correlation): it only draws random numbers and renders a phantom.  Both
 * the FP64 oracle (oracle/) and the CUDA library (paper_2603_15285_b200/) consume the
 * float32 volumes it writes, so the two sides see bit-identical inputs.
 *
 * Workload recipe (shaped like PAPER.md P:941-949, which uses
 * the EMD-3228 ribosome, unavailable here):
 *   reference h : 32 anisotropic Gaussian blobs, centres uniform in the ball of radius 0.6
 *                 (half-box units), principal widths U[0.05,0.2], Haar-random orientation,
 *                 amplitude U[0.5,1], rendered analytically at voxel centres
 *                 y = (v - c)/(N/2), c = (N-1)/2.
 *   particle p  : f = S_t(g o h) + eta  (P:945 with the App. C shift, reading C17):
 *                 f(x) = h(g^T (x - c - t)/(N/2)), g Haar (normalised 4-D Gaussian
 *                 quaternion), t zero / U[-s,s]^3 / fixed; eta ~ N(0, P_ref/SNR) i.i.d.,
 *                 P_ref = mean over the N^3 box of h^2 (reading C21, linear SNR).
 * Random numbers: Philox4x32-10, key = (seed lo, seed hi), counter = (a, b, c, stream).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

enum { STREAM_REF = 0x100, STREAM_ROT = 0x200, STREAM_SHIFT = 0x300, STREAM_NOISE = 0x400 };

static void philox4x32_10(const uint32_t ctr_in[4], uint64_t seed, uint32_t out[4]) {
  uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)PHILOX_M0 * c[0];
    uint64_t p1 = (uint64_t)PHILOX_M1 * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += PHILOX_W0; k1 += PHILOX_W1;
  }
  memcpy(out, c, sizeof(c));
}

/* open-interval uniform (0,1) */
static double u01(uint32_t x) { return ((double)x + 0.5) * (1.0 / 4294967296.0); }

static void uniforms4(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t stream, double u[4]) {
  uint32_t ctr[4] = {a, b, c, stream}, o[4];
  philox4x32_10(ctr, seed, o);
  for (int i = 0; i < 4; ++i) u[i] = u01(o[i]);
}

static void normals4(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t stream, double z[4]) {
  double u[4];
  uniforms4(seed, a, b, c, stream, u);
  for (int i = 0; i < 4; i += 2) {
    double rad = sqrt(-2.0 * log(u[i]));
    z[i] = rad * cos(2.0 * M_PI * u[i + 1]);
    z[i + 1] = rad * sin(2.0 * M_PI * u[i + 1]);
  }
}

/* rotation matrix (row-major) of a unit quaternion (w,x,y,z) */
static void quat_to_matrix(const double q_in[4], double R[9]) {
  double n = sqrt(q_in[0] * q_in[0] + q_in[1] * q_in[1] + q_in[2] * q_in[2] + q_in[3] * q_in[3]);
  double w = q_in[0] / n, x = q_in[1] / n, y = q_in[2] / n, z = q_in[3] / n;
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

/* blobs: [nblobs][10] = mu(3), Sinv (xx,yy,zz,xy,xz,yz), amp */
void gen_reference_blobs(uint64_t seed, int nblobs, double* blobs) {
  for (int b = 0; b < nblobs; ++b) {
    double z0[4], u1[4], q[4], u3[4];
    normals4(seed, (uint32_t)b, 0, 0, STREAM_REF, z0);
    uniforms4(seed, (uint32_t)b, 1, 0, STREAM_REF, u1);
    normals4(seed, (uint32_t)b, 2, 0, STREAM_REF, q);
    uniforms4(seed, (uint32_t)b, 3, 0, STREAM_REF, u3);
    double dn = sqrt(z0[0] * z0[0] + z0[1] * z0[1] + z0[2] * z0[2]);
    double rad = 0.6 * cbrt(u1[0]);
    double* o = blobs + 10 * b;
    for (int i = 0; i < 3; ++i) o[i] = rad * z0[i] / dn;
    double sig[3];
    for (int i = 0; i < 3; ++i) sig[i] = 0.05 + 0.15 * u1[1 + i];
    double Q[9];
    quat_to_matrix(q, Q);
    double S[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0;
        for (int k = 0; k < 3; ++k) s += Q[3 * i + k] * Q[3 * j + k] / (sig[k] * sig[k]);
        S[i][j] = s;
      }
    o[3] = S[0][0]; o[4] = S[1][1]; o[5] = S[2][2]; o[6] = S[0][1]; o[7] = S[0][2]; o[8] = S[1][2];
    o[9] = 0.5 + 0.5 * u3[0];
  }
}

/* Transform blobs by x -> R x + (shift in half-box units): mu' = R mu + s, Sinv' = R Sinv R^T. */
static void transform_blobs(const double* in, int nb, const double* R, const double* s, double* out) {
  for (int b = 0; b < nb; ++b) {
    const double* p = in + 10 * b;
    double* o = out + 10 * b;
    double S[3][3] = {{p[3], p[6], p[7]}, {p[6], p[4], p[8]}, {p[7], p[8], p[5]}};
    double T[3][3], U[3][3];
    for (int i = 0; i < 3; ++i) {
      double m = 0;
      for (int k = 0; k < 3; ++k) m += R[3 * i + k] * p[k];
      o[i] = m + s[i];
    }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double v = 0;
        for (int k = 0; k < 3; ++k) v += R[3 * i + k] * S[k][j];
        T[i][j] = v;
      }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double v = 0;
        for (int k = 0; k < 3; ++k) v += T[i][k] * R[3 * j + k];
        U[i][j] = v;
      }
    o[3] = U[0][0]; o[4] = U[1][1]; o[5] = U[2][2]; o[6] = U[0][1]; o[7] = U[0][2]; o[8] = U[1][2];
    o[9] = p[9];
  }
}

/* inverse of a symmetric 3x3 given as (xx,yy,zz,xy,xz,yz): returns diagonal of the inverse */
static void sym_inv_diag(const double* s, double d[3]) {
  double a = s[0], b = s[1], c = s[2], xy = s[3], xz = s[4], yz = s[5];
  double det = a * (b * c - yz * yz) - xy * (xy * c - yz * xz) + xz * (xy * yz - b * xz);
  d[0] = (b * c - yz * yz) / det;
  d[1] = (a * c - xz * xz) / det;
  d[2] = (a * b - xy * xy) / det;
}

/* Render sum of blobs at voxel centres (accumulating into a double buffer). Returns mean square. */
static double render(const double* blobs, int nb, int N, double* acc, float* vol) {
  const double c = 0.5 * (N - 1), hb = 0.5 * N;
  const size_t n3 = (size_t)N * N * N;
  for (size_t i = 0; i < n3; ++i) acc[i] = 0.0;
  const double QCUT = 50.0; /* exp(-25) ~ 1.4e-11: below float resolution of the O(1) sums */
  for (int b = 0; b < nb; ++b) {
    const double* p = blobs + 10 * b;
    double cov[3];
    sym_inv_diag(p + 3, cov);
    int lo[3], hi[3];
    for (int i = 0; i < 3; ++i) {
      double ext = sqrt(QCUT * cov[i]);
      lo[i] = (int)floor((p[i] - ext) * hb + c);
      hi[i] = (int)ceil((p[i] + ext) * hb + c);
      if (lo[i] < 0) lo[i] = 0;
      if (hi[i] > N - 1) hi[i] = N - 1;
    }
    for (int z = lo[2]; z <= hi[2]; ++z) {
      double dz = (z - c) / hb - p[2];
      for (int y = lo[1]; y <= hi[1]; ++y) {
        double dy = (y - c) / hb - p[1];
        double* row = acc + ((size_t)z * N + y) * N;
        for (int x = lo[0]; x <= hi[0]; ++x) {
          double dx = (x - c) / hb - p[0];
          double q = p[3] * dx * dx + p[4] * dy * dy + p[5] * dz * dz +
                     2.0 * (p[6] * dx * dy + p[7] * dx * dz + p[8] * dy * dz);
          if (q < QCUT) row[x] += p[9] * exp(-0.5 * q);
        }
      }
    }
  }
  double ms = 0.0;
  for (size_t i = 0; i < n3; ++i) {
    ms += acc[i] * acc[i];
    if (vol) vol[i] = (float)acc[i];
  }
  return ms / (double)n3;
}

/* Render reference (R=NULL,t=NULL) or a transformed copy f(x) = h(R^T (x - c - t)/(N/2)).
   Returns mean over the box of the rendered (noise-free) values squared. */
double gen_render(const double* blobs, int nblobs, int N, const double* R9, const double* t3, float* vol) {
  double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, z[3] = {0, 0, 0};
  double s[3];
  const double* R = R9 ? R9 : I;
  const double* t = t3 ? t3 : z;
  for (int i = 0; i < 3; ++i) s[i] = t[i] / (0.5 * N);
  double* tb = (double*)malloc(sizeof(double) * 10 * (size_t)nblobs);
  double* acc = (double*)malloc(sizeof(double) * (size_t)N * N * N);
  transform_blobs(blobs, nblobs, R, s, tb);
  double ms = render(tb, nblobs, N, acc, vol);
  free(acc);
  free(tb);
  return ms;
}

/* shift_mode: 0 zero, 1 uniform U[-shift_max, shift_max]^3, 2 fixed (fixed_shift) */
void gen_particle_pose(uint64_t seed, int64_t p, int shift_mode, double shift_max, const double* fixed_shift,
                       double* R9, double* t3) {
  double q[4];
  normals4(seed, (uint32_t)(p & 0xffffffff), (uint32_t)((uint64_t)p >> 32), 0, STREAM_ROT, q);
  quat_to_matrix(q, R9);
  if (shift_mode == 1) {
    double u[4];
    uniforms4(seed, (uint32_t)(p & 0xffffffff), (uint32_t)((uint64_t)p >> 32), 0, STREAM_SHIFT, u);
    for (int i = 0; i < 3; ++i) t3[i] = shift_max * (2.0 * u[i] - 1.0);
  } else if (shift_mode == 2) {
    for (int i = 0; i < 3; ++i) t3[i] = fixed_shift[i];
  } else {
    t3[0] = t3[1] = t3[2] = 0.0;
  }
}

void gen_add_noise(uint64_t seed, int64_t p, int N, double sigma, float* vol) {
  const size_t n3 = (size_t)N * N * N;
  for (size_t v = 0; v < n3; v += 4) {
    double z[4];
    normals4(seed, (uint32_t)(p & 0xffffffff), (uint32_t)((uint64_t)p >> 32), (uint32_t)(v / 4), STREAM_NOISE, z);
    for (size_t i = 0; i < 4 && v + i < n3; ++i) vol[v + i] = (float)((double)vol[v + i] + sigma * z[i]);
  }
}

typedef struct {
  uint64_t seed;
  const double* blobs;
  int nblobs, N, shift_mode;
  int64_t first, B;
  double sigma, shift_max;
  const double* fixed_shift;
  float* vols;
  double* truth;
  int tid, nthreads;
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  const size_t n3 = (size_t)j->N * j->N * j->N;
  double* acc = (double*)malloc(sizeof(double) * n3);
  double* tb = (double*)malloc(sizeof(double) * 10 * (size_t)j->nblobs);
  for (int64_t i = j->tid; i < j->B; i += j->nthreads) {
    int64_t p = j->first + i;
    double R[9], t[3], s[3];
    gen_particle_pose(j->seed, p, j->shift_mode, j->shift_max, j->fixed_shift, R, t);
    for (int k = 0; k < 3; ++k) s[k] = t[k] / (0.5 * j->N);
    transform_blobs(j->blobs, j->nblobs, R, s, tb);
    float* vol = j->vols + (size_t)i * n3;
    render(tb, j->nblobs, j->N, acc, vol);
    if (j->sigma > 0) gen_add_noise(j->seed, p, j->N, j->sigma, vol);
    if (j->truth) {
      memcpy(j->truth + 12 * i, R, sizeof(R));
      memcpy(j->truth + 12 * i + 9, t, sizeof(t));
    }
  }
  free(tb);
  free(acc);
  return NULL;
}

/* Particles first..first+B-1 of the stream `seed`. snr <= 0 or inf => noise-free.
   p_ref: mean square of the noise-free reference (reading C21).  truth [B][12] = R(9), t(3).
   Returns the noise sigma used. */
double gen_particles(uint64_t seed, const double* blobs, int nblobs, int N, int64_t first, int64_t B, double snr,
                     double p_ref, int shift_mode, double shift_max, const double* fixed_shift, float* vols,
                     double* truth, int nthreads) {
  double sigma = (snr > 0 && isfinite(snr)) ? sqrt(p_ref / snr) : 0.0;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  job_t jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    job_t jb = {seed, blobs, nblobs, N, shift_mode, first, B, sigma, shift_max, fixed_shift, vols, truth, t, nthreads};
    jobs[t] = jb;
    pthread_create(&th[t], NULL, worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  return sigma;
}
