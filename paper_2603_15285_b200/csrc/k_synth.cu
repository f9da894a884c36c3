// k_synth.cu -- matcha_synth_particles: the seeded synthetic workload generated on the device,
// so bench inputs at STA scale (c4: 100k particles) need no host rendering.  Test/bench infrastructure, not the
// method: Philox4x32-10 random numbers and the Gaussian-blob phantom of DESIGN.md "Input recipe", the same counter
// layout and arithmetic order as gen/gen.c (each side implements the same counter-based generator; the CUDA
// path's volumes are never fed to the oracle).
//   reference: 32 anisotropic blobs (Philox key 0x5EED, stream 0x100), rendered at voxel centres x = (v - c)/(N/2);
//   particle p: Haar rotation (4 normals, stream 0x200), shift U[-s, s]^3 (stream 0x300), blobs rendered at the
//   rotated/shifted positions, + N(0, P_ref/SNR) noise (stream 0x400, Box-Muller), P_ref = mean square of the
//   reference (reading C21).
#include <cmath>

#include "common.cuh"

namespace matcha {

namespace {

constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u, kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;
constexpr uint32_t kStreamRef = 0x100, kStreamRot = 0x200, kStreamShift = 0x300, kStreamNoise = 0x400;
constexpr uint64_t kRefSeed = 0x5EED;
constexpr int kBlobs = 32;
constexpr double kQCut = 50.0;

__device__ void philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t seed, uint32_t out[4]) {
  uint32_t c[4] = {c0, c1, c2, c3};
  uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)kM0 * c[0], p1 = (uint64_t)kM1 * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += kW0;
    k1 += kW1;
  }
  for (int i = 0; i < 4; ++i) out[i] = c[i];
}
__device__ void uniforms4(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t st, double u[4]) {
  uint32_t o[4];
  philox(a, b, c, st, seed, o);
  for (int i = 0; i < 4; ++i) u[i] = ((double)o[i] + 0.5) * (1.0 / 4294967296.0);
}
__device__ void normals4(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t st, double z[4]) {
  double u[4];
  uniforms4(seed, a, b, c, st, u);
  for (int i = 0; i < 4; i += 2) {
    const double rad = sqrt(-2.0 * log(u[i]));
    z[i] = rad * cos(2.0 * kPi * u[i + 1]);
    z[i + 1] = rad * sin(2.0 * kPi * u[i + 1]);
  }
}
__device__ void quat_to_matrix(const double q[4], double R[9]) {
  const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

// the reference blobs: [kBlobs][10] = mu(3), Sinv (xx, yy, zz, xy, xz, yz), amp
__global__ void k_ref_blobs(double* __restrict__ blobs) {
  const int b = threadIdx.x;
  if (b >= kBlobs) return;
  double z0[4], u1[4], q[4], u3[4];
  normals4(kRefSeed, (uint32_t)b, 0, 0, kStreamRef, z0);
  uniforms4(kRefSeed, (uint32_t)b, 1, 0, kStreamRef, u1);
  normals4(kRefSeed, (uint32_t)b, 2, 0, kStreamRef, q);
  uniforms4(kRefSeed, (uint32_t)b, 3, 0, kStreamRef, u3);
  const double dn = sqrt(z0[0] * z0[0] + z0[1] * z0[1] + z0[2] * z0[2]);
  const double rad = 0.6 * cbrt(u1[0]);
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

// per particle: pose (truth) and the transformed blobs mu' = R mu + t/(N/2), Sinv' = R Sinv R^T
// particle index pi < 0 renders the reference itself (identity pose)
__global__ void k_pose_blobs(const double* __restrict__ ref, uint64_t seed, int64_t first, int64_t B, int N,
                             double shift_max, double* __restrict__ tblobs, double* __restrict__ truth) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= B) return;
  double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, t[3] = {0, 0, 0};
  if (first >= 0) {
    const int64_t p = first + i;
    double q[4];
    normals4(seed, (uint32_t)(p & 0xffffffff), (uint32_t)((uint64_t)p >> 32), 0, kStreamRot, q);
    quat_to_matrix(q, R);
    if (shift_max > 0) {
      double u[4];
      uniforms4(seed, (uint32_t)(p & 0xffffffff), (uint32_t)((uint64_t)p >> 32), 0, kStreamShift, u);
      for (int k = 0; k < 3; ++k) t[k] = shift_max * (2.0 * u[k] - 1.0);
    }
  }
  if (truth) {
    for (int k = 0; k < 9; ++k) truth[i * 12 + k] = R[k];
    for (int k = 0; k < 3; ++k) truth[i * 12 + 9 + k] = t[k];
  }
  double s[3];
  for (int k = 0; k < 3; ++k) s[k] = t[k] / (0.5 * N);
  for (int b = 0; b < kBlobs; ++b) {
    const double* p = ref + 10 * b;
    double* o = tblobs + (i * kBlobs + b) * 10;
    const double S[3][3] = {{p[3], p[6], p[7]}, {p[6], p[4], p[8]}, {p[7], p[8], p[5]}};
    double T[3][3], U[3][3];
    for (int r = 0; r < 3; ++r) {
      double m = 0;
      for (int k = 0; k < 3; ++k) m += R[3 * r + k] * p[k];
      o[r] = m + s[r];
    }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double v = 0;
        for (int k = 0; k < 3; ++k) v += R[3 * r + k] * S[k][c];
        T[r][c] = v;
      }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double v = 0;
        for (int k = 0; k < 3; ++k) v += T[r][k] * R[3 * c + k];
        U[r][c] = v;
      }
    o[3] = U[0][0]; o[4] = U[1][1]; o[5] = U[2][2]; o[6] = U[0][1]; o[7] = U[0][2]; o[8] = U[1][2];
    o[9] = p[9];
  }
}

// one thread per 4 consecutive voxels of particle blockIdx.y: the blob sum (in blob order, q < QCUT as gen.c's
// bounding-box loops), rounded to float, then the noise of the same 4-voxel Philox counter added in double and
// rounded again (gen_add_noise)
__global__ void __launch_bounds__(256) k_render(const double* __restrict__ tblobs, uint64_t seed, int64_t first,
                                                int N, const double* __restrict__ sigma_p, float* __restrict__ vols,
                                                double* __restrict__ sq) {
  __shared__ double bl[kBlobs * 10];
  const int64_t i = blockIdx.y;
  for (int t = threadIdx.x; t < kBlobs * 10; t += blockDim.x) bl[t] = tblobs[i * kBlobs * 10 + t];
  __syncthreads();
  const int64_t n3 = (int64_t)N * N * N;
  const int64_t v0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (v0 >= n3) return;
  const double c = 0.5 * (N - 1), hb = 0.5 * N;
  double acc[4];
  for (int q = 0; q < 4; ++q) {
    const int64_t v = v0 + q;
    acc[q] = 0.0;
    if (v >= n3) continue;
    const int x = (int)(v % N), y = (int)((v / N) % N), z = (int)(v / ((int64_t)N * N));
    for (int b = 0; b < kBlobs; ++b) {
      const double* p = bl + 10 * b;
      const double dx = (x - c) / hb - p[0], dy = (y - c) / hb - p[1], dz = (z - c) / hb - p[2];
      const double qq = p[3] * dx * dx + p[4] * dy * dy + p[5] * dz * dz +
                        2.0 * (p[6] * dx * dy + p[7] * dx * dz + p[8] * dy * dz);
      if (qq < kQCut) acc[q] += p[9] * exp(-0.5 * qq);
    }
  }
  if (sq) {  // the reference: squares for P_ref
    for (int q = 0; q < 4; ++q)
      if (v0 + q < n3) sq[v0 + q] = acc[q] * acc[q];
    return;
  }
  float* vol = vols + i * n3;
  const double sigma = *sigma_p;
  double zn[4] = {0, 0, 0, 0};
  if (sigma > 0) {
    const int64_t p = first + i;
    normals4(seed, (uint32_t)(p & 0xffffffff), (uint32_t)((uint64_t)p >> 32), (uint32_t)(v0 / 4), kStreamNoise, zn);
  }
  for (int q = 0; q < 4; ++q)
    if (v0 + q < n3) {
      const float f = (float)acc[q];
      vol[v0 + q] = sigma > 0 ? (float)((double)f + sigma * zn[q]) : f;
    }
}

// P_ref = mean of sq (fixed-order single-CTA reduction), sigma = sqrt(P_ref / snr) (0 when snr <= 0 or infinite)
__global__ void __launch_bounds__(256) k_sigma(const double* __restrict__ sq, int64_t n, double snr,
                                               double* __restrict__ out) {
  __shared__ double red[256];
  double s = 0;
  for (int64_t i = threadIdx.x; i < n; i += 256) s += sq[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double pref = red[0] / (double)n;
    out[0] = (snr > 0 && isfinite(snr)) ? sqrt(pref / snr) : 0.0;
    out[1] = pref;
  }
}

}  // namespace

size_t synth_workspace_bytes(int N, int64_t B) {
  return sizeof(double) * ((size_t)kBlobs * 10 * (B + 2) + (size_t)N * N * N + 8);
}

cudaError_t launch_synth_particles(uint64_t seed, int64_t first, int64_t B, int N, double snr, double shift_max,
                                   float* vols, double* truth, void* ws, cudaStream_t s) {
  double* ref = reinterpret_cast<double*>(ws);
  double* sig = ref + kBlobs * 10;              // [sigma, P_ref]
  double* rblob = sig + 8;                      // reference "pose blobs" (identity)
  double* sq = rblob + kBlobs * 10;             // [N^3]
  double* tb = sq + (int64_t)N * N * N;         // [B][kBlobs][10]
  k_ref_blobs<<<1, kBlobs, 0, s>>>(ref);
  k_pose_blobs<<<1, 32, 0, s>>>(ref, seed, -1, 1, N, 0.0, rblob, nullptr);
  const int64_t n3 = (int64_t)N * N * N, nt = (n3 / 4 + 255) / 256;
  k_render<<<dim3((unsigned)nt, 1), 256, 0, s>>>(rblob, seed, 0, N, nullptr, nullptr, sq);
  k_sigma<<<1, 256, 0, s>>>(sq, n3, snr, sig);
  if (B > 0) {
    k_pose_blobs<<<(unsigned)((B + 127) / 128), 128, 0, s>>>(ref, seed, first, B, N, shift_max, tb, truth);
    for (int64_t b0 = 0; b0 < B; b0 += 65535) {
      const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
      k_render<<<dim3((unsigned)nt, (unsigned)nb), 256, 0, s>>>(tb + b0 * kBlobs * 10, seed, first + b0, N, sig,
                                                                vols + b0 * n3, nullptr);
    }
  }
  return cudaGetLastError();
}

}  // namespace matcha
