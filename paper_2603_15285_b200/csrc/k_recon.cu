// k_recon.cu -- SURVEY f4: the subtomogram-averaging reference update that follows an alignment pass.
//
// PAPER.md P:1184 (Matcha "estimates both rotations and translations using the same half-set split as RELION") and
// P:1202 ("in practice the reference template is itself unknown and must be iteratively estimated from the data");
// reading C28: with the generative model f_p(x) = h(g_p^T (x - c - t_p) + c) (reading C17) the aligned particle in
// the reference frame is f_p(g_p (y - c) + c + t_p), and the half maps are the plain sums
//   S_{k,s}(y) = sum_{p : class(p) = k, (first + p) mod 2 = s} f_p(g_p (y - c) + c + t_p)
// (trilinear, zero outside; reading C5), with the counts n_{k,s}; the average is S / n.  Multi-GPU: every rank sums
// its shard, one all-reduce (the only N^3 collective of the domain), then the division.
//
// B200 mapping: a warp per (class, half) compacts its particle indices in increasing order (ballot), then one CTA per
// (8 x 8 x 4 voxel tile, class, half), each thread one voxel, walks its list in chunks of 32 poses staged in shared
// memory (fixed summation order: deterministic, no atomics), the rotated tile footprints read through L1.
#include <algorithm>

#include "common.cuh"

namespace matcha {

namespace {

// per particle: R (row-major) and t, from the pose row {alpha, beta, gamma, tx, ty, tz, ...}
template <typename T>
__global__ void k_pose_mats(const T* __restrict__ poses, int pstride, int64_t B, T* __restrict__ Rt) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= B) return;
  const T* e = poses + p * pstride;
  double sa, ca, sb, cb, sg, cg;
  sincos((double)e[0], &sa, &ca);
  sincos((double)e[1], &sb, &cb);
  sincos((double)e[2], &sg, &cg);
  // g = r_z(a) r_y(b) r_z(g)  (Eq. 3)
  const double R[9] = {ca * cb * cg - sa * sg, -ca * cb * sg - sa * cg, ca * sb,
                       sa * cb * cg + ca * sg, -sa * cb * sg + ca * cg, sa * sb,
                       -sb * cg,               sb * sg,                 cb};
  T* o = Rt + p * 12;
  for (int k = 0; k < 9; ++k) o[k] = (T)R[k];
  o[9] = e[3];
  o[10] = e[4];
  o[11] = e[5];
}

constexpr int kTx = 8, kTy = 8, kTz = 4;
constexpr int kChunk = 32;  // particles whose poses are staged in shared memory at a time

// per (class, half): the particle indices in increasing order (one warp per list, ballot compaction: deterministic)
template <typename T>
__global__ void k_recon_lists(const T* __restrict__ poses, int pstride, int ccol, int ncls, int64_t B, int64_t first,
                              int* __restrict__ lists, int* __restrict__ counts) {
  const int list = blockIdx.x;  // class * 2 + half
  if (list >= 2 * ncls) return;
  const int cls = list >> 1, half = list & 1, lane = threadIdx.x;
  int n = 0;
  for (int64_t p0 = 0; p0 < B; p0 += 32) {
    const int64_t p = p0 + lane;
    bool take = false;
    if (p < B) {
      const int k = ccol >= 0 ? (int)poses[p * pstride + ccol] : 0;
      take = k == cls && (int)((first + p) & 1) == half;
    }
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (take) lists[(int64_t)list * B + n + __popc(m & ((1u << lane) - 1))] = (int)p;
    n += __popc(m);
  }
  if (lane == 0) counts[list] = n;
}

template <typename T>
__global__ void __launch_bounds__(kTx * kTy * kTz) k_backproject(const float* __restrict__ vols, int64_t B, int N,
                                                                 const T* __restrict__ Rt,
                                                                 const int* __restrict__ lists,
                                                                 const int* __restrict__ counts,
                                                                 T* __restrict__ sums) {
  __shared__ T sRt[kChunk][12];
  __shared__ int sp[kChunk];
  const int ntx = N / kTx, nty = N / kTy;
  const int tile = blockIdx.x, tx = tile % ntx, ty = (tile / ntx) % nty, tz = tile / (ntx * nty);
  const int x = tx * kTx + (threadIdx.x % kTx), y = ty * kTy + (threadIdx.x / kTx) % kTy,
            z = tz * kTz + threadIdx.x / (kTx * kTy);
  const T c = T(0.5) * (T)(N - 1);
  const T ux = (T)x - c, uy = (T)y - c, uz = (T)z - c;
  const int64_t n3 = (int64_t)N * N * N;
  const int* lst = lists + (int64_t)blockIdx.y * B;
  const int cnt = counts[blockIdx.y];
  T acc = T(0);
  for (int j0 = 0; j0 < cnt; j0 += kChunk) {
    const int nj = min(kChunk, cnt - j0);
    __syncthreads();
    for (int t = threadIdx.x; t < nj * 12; t += blockDim.x) {
      const int j = t / 12, q = t - j * 12;
      sRt[j][q] = Rt[(int64_t)lst[j0 + j] * 12 + q];
    }
    for (int t = threadIdx.x; t < nj; t += blockDim.x) sp[t] = lst[j0 + t];
    __syncthreads();
    for (int j = 0; j < nj; ++j) {
      const T* m = sRt[j];
      const T qx = fma(m[0], ux, fma(m[1], uy, m[2] * uz)) + c + m[9];  // g (y - c) + c + t
      const T qy = fma(m[3], ux, fma(m[4], uy, m[5] * uz)) + c + m[10];
      const T qz = fma(m[6], ux, fma(m[7], uy, m[8] * uz)) + c + m[11];
      const T fx0 = floor(qx), fy0 = floor(qy), fz0 = floor(qz);
      const int x0 = (int)fx0, y0 = (int)fy0, z0 = (int)fz0;
      const T fx = qx - fx0, fy = qy - fy0, fz = qz - fz0;
      const float* v = vols + (int64_t)sp[j] * n3;
      T cc[2][2][2];
#pragma unroll
      for (int dz = 0; dz < 2; ++dz)
#pragma unroll
        for (int dy = 0; dy < 2; ++dy)
#pragma unroll
          for (int dx = 0; dx < 2; ++dx) {
            const int xx = x0 + dx, yy = y0 + dy, zz = z0 + dz;
            const bool in = (unsigned)xx < (unsigned)N && (unsigned)yy < (unsigned)N && (unsigned)zz < (unsigned)N;
            cc[dz][dy][dx] = in ? (T)__ldg(v + ((int64_t)zz * N + yy) * N + xx) : T(0);
          }
      const T c00 = fma(fx, cc[0][0][1] - cc[0][0][0], cc[0][0][0]);
      const T c01 = fma(fx, cc[0][1][1] - cc[0][1][0], cc[0][1][0]);
      const T c10 = fma(fx, cc[1][0][1] - cc[1][0][0], cc[1][0][0]);
      const T c11 = fma(fx, cc[1][1][1] - cc[1][1][0], cc[1][1][0]);
      const T c0 = fma(fy, c01 - c00, c00);
      const T c1 = fma(fy, c11 - c10, c10);
      acc += fma(fz, c1 - c0, c0);
    }
  }
  sums[(int64_t)blockIdx.y * n3 + ((int64_t)z * N + y) * N + x] = acc;
}

}  // namespace

template <typename T>
cudaError_t launch_reconstruct(const float* vols, int64_t B, int N, const T* poses, int pstride, int ccol, int ncls,
                               int64_t first, T* Rt, T* sums, int* counts, cudaStream_t s) {
  if (N % kTx || N % kTz) return cudaErrorInvalidValue;
  int* lists = reinterpret_cast<int*>(Rt + 12 * (B > 0 ? B : 1));  // [2 ncls][B] behind the pose matrices
  if (B > 0) {
    k_pose_mats<T><<<(unsigned)((B + 127) / 128), 128, 0, s>>>(poses, pstride, B, Rt);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  k_recon_lists<T><<<(unsigned)(2 * ncls), 32, 0, s>>>(poses, pstride, ccol, ncls, B, first, lists, counts);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int tiles = (N / kTx) * (N / kTy) * (N / kTz);
  k_backproject<T><<<dim3((unsigned)tiles, (unsigned)(2 * ncls)), kTx * kTy * kTz, 0, s>>>(vols, B, N, Rt, lists,
                                                                                           counts, sums);
  return cudaGetLastError();
}

size_t reconstruct_workspace_bytes(int64_t B, int ncls, size_t rsz) {
  const int64_t b = B > 0 ? B : 1;
  return rsz * 12 * (size_t)b + sizeof(int) * 2 * (size_t)ncls * (size_t)b + 64;
}

template cudaError_t launch_reconstruct<float>(const float*, int64_t, int, const float*, int, int, int, int64_t, float*,
                                               float*, int*, cudaStream_t);
template cudaError_t launch_reconstruct<double>(const float*, int64_t, int, const double*, int, int, int, int64_t,
                                                double*, double*, int*, cudaStream_t);

}  // namespace matcha
