// k_corr_tc.cu -- stage 2 on the 5th-generation tensor cores (tcgen05, TMEM accumulators), FP32 handles.
//
// M^l_mn = sum_i w_i f_lm(r_i) conj(h_ln(r_i))  (reading C2) is, per degree l,
// the complex GEMM [(particles x (l+1)) x R] . [R x (2l+1)].  It is run as ONE real GEMM per (l, 128-row tile)
// with interleaved complex operands, so neither input nor output is reshuffled:
//   A[row = (p, m)][k = 2r + c]   = F[p][lm(l,m)][r].{re,im}                  (the F rows as stored)
//   B[col = 2nn + c'][k = 2r + c] = [[Hc.re, -Hc.im], [Hc.im, Hc.re]]  with Hc = w_r conj(h_{l,nn-l}(r))
//   D[row][col]                   = M[p][l(l+1)(4l-1)/6 + m(2l+1)].{re,im} of nn  (the M rows as stored)
// kind::tf32 with a 3-pass split (x = hi + lo, hi = x with the low 13 mantissa bits cleared):
//   D = A_hi B_hi + A_hi B_lo + A_lo B_hi   (relative error ~2^-21, i.e. FP32-level; lo*lo dropped).
// Operands: K-major, SWIZZLE_NONE canonical layout (8-row x 16-byte core matrices; SBO = 128 B between 8-row
// groups, LBO = rows*16 B between 16-byte K chunks), staged in shared memory by the CTA's threads (the hi/lo
// split happens on the way in); one elected thread issues the 3 x (2R/8) tcgen05.mma; tcgen05.commit arrives
// on an mbarrier; the 4 warps read the 128 x N fp32 accumulator out of TMEM with tcgen05.ld (one TMEM lane per
// row) and store the complex rows of M directly.  Persistent CTAs walk tiles l-major so B is rebuilt only
// when l changes.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace matcha {

namespace {

constexpr int kTM = 128;          // UMMA_M (rows per tile, one TMEM lane per row)
constexpr int kTCThreads = 512;   // 16 warps: warp w reads TMEM lane quarter w % 4, column slice w / 4

__host__ __device__ inline int tile_n(int l) { return (2 * (2 * l + 1) + 15) / 16 * 16; }  // UMMA_N, % 16 == 0
__host__ __device__ inline int tmem_cols(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : 256; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, SWIZZLE_NONE shared-memory matrix descriptor (sm_100 version 1)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}

// instruction descriptor: kind::tf32, D fp32, A/B tf32 K-major, M = 128, N
__host__ __device__ inline uint32_t make_idesc(int N) {
  uint32_t d = 0;
  d |= 1u << 4;                    // c_format = F32
  d |= 2u << 7;                    // a_format = TF32
  d |= 2u << 10;                   // b_format = TF32
  d |= (uint32_t)(N >> 3) << 17;   // n_dim
  d |= (uint32_t)(kTM >> 4) << 24; // m_dim
  return d;
}

// element (row i, k) of a K-major SWIZZLE_NONE operand with `rows` rows: byte offset
__device__ __forceinline__ uint32_t kmaj_off(int i, int k, int rows) {
  return (uint32_t)((i & 7) * 16 + (i >> 3) * 128 + (k & 3) * 4 + (k >> 2) * rows * 16);
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

struct TileMap {
  int l, row0;
};

// tile t -> (l, first row) with tiles enumerated l-major: l has ceil(B (l+1) / 128) tiles
__device__ __forceinline__ TileMap tile_of(int64_t t, int64_t B, int L) {
  TileMap m{-1, 0};
  for (int l = 0; l <= L; ++l) {
    const int64_t nt = (B * (l + 1) + kTM - 1) / kTM;
    if (t < nt) {
      m.l = l;
      m.row0 = (int)(t * kTM);
      return m;
    }
    t -= nt;
  }
  return m;
}

__global__ void __launch_bounds__(kTCThreads, 1)
    k_corr_tc(const float2* __restrict__ F, const float2* __restrict__ H, int64_t B, int L, int Lmax, int R,
              int64_t ntiles, float2* __restrict__ M) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int K = 2 * R;                       // real K (multiple of 8: R % 4 == 0)
  const int NMAX = tile_n(L);
  // layout: A_hi, A_lo [128 x K], B_hi, B_lo [NMAX x K] (fp32 words), then mbarrier + tmem slot
  float* Ahi = (float*)smem;
  float* Alo = Ahi + kTM * K;
  float* Bhi = Alo + kTM * K;
  float* Blo = Bhi + NMAX * K;
  float* Dst = Blo + NMAX * K;               // [128][NMAX + 1] fp32 staging of the accumulator tile
  uint64_t* mbar = (uint64_t*)(Dst + ((kTM * (NMAX + 1) + 3) & ~3));  // 16-byte aligned
  uint32_t* tslot = (uint32_t*)(mbar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncf = ncoef(Lmax);
  const uint32_t ncols = (uint32_t)tmem_cols(NMAX);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tslot;
  uint32_t phase = 0;
  int cur_l = -1;

  // contiguous tile ranges per CTA: consecutive tiles share l, so B is rebuilt about once per CTA
  const int64_t t_begin = ntiles * blockIdx.x / gridDim.x, t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  for (int64_t t = t_begin; t < t_end; ++t) {
    const TileMap tm = tile_of(t, B, L);
    const int l = tm.l, w = 2 * l + 1, N = tile_n(l);
    const int64_t rows_l = B * (l + 1);
    // B operand for degree l (rebuilt only when l changes)
    if (l != cur_l) {
      const float2* Hl = H + (int64_t)lm_index(l, 0) * R;
      for (int e = tid; e < (N / 2) * R; e += kTCThreads) {
        const int col2 = e / R, r = e - col2 * R;  // col2 = output complex column pair index nn (padded to N/2)
        const int nn = col2;
        float hre = 0.f, him = 0.f;
        if (nn < w) {
          const int n = nn - l;
          const float rr = (float)r + 0.5f, wr = rr * rr;
          const float2 h = Hl[(size_t)abs(n) * R + r];
          if (n >= 0) {
            hre = wr * h.x;
            him = -wr * h.y;
          } else {
            const float sg = (n & 1) ? -1.f : 1.f;
            hre = sg * wr * h.x;
            him = sg * wr * h.y;
          }
        }
        // columns 2nn (Re out) and 2nn+1 (Im out); k = 2r (Re in), 2r+1 (Im in)
        if (2 * nn < N) {
          const float v[4] = {hre, -him, him, hre};  // (col 2nn: k 2r, k 2r+1), (col 2nn+1: k 2r, k 2r+1)
          const int cols[4] = {2 * nn, 2 * nn, 2 * nn + 1, 2 * nn + 1};
          const int ks[4] = {2 * r, 2 * r + 1, 2 * r, 2 * r + 1};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float hi = tf32_hi(v[q]);
            const uint32_t off = kmaj_off(cols[q], ks[q], N);
            *(float*)((unsigned char*)Bhi + off) = hi;
            *(float*)((unsigned char*)Blo + off) = v[q] - hi;
          }
        }
      }
      cur_l = l;
    }
    // A operand: 128 rows (p, m) of F, interleaved complex along k
    for (int e = tid; e < kTM * (K / 4); e += kTCThreads) {
      const int i = e / (K / 4), k4 = e - i * (K / 4);
      const int64_t row = tm.row0 + i;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < rows_l) {
        const int64_t p = row / (l + 1);
        const int m = (int)(row - p * (l + 1));
        v = __ldg(reinterpret_cast<const float4*>(F + (p * ncf + lm_index(l, m)) * R) + k4);
      }
      const float vv[4] = {v.x, v.y, v.z, v.w};
      const uint32_t off = kmaj_off(i, 4 * k4, kTM);  // 4 consecutive k = one 16-byte chunk
      float4 hi, lo;
      hi.x = tf32_hi(vv[0]);
      hi.y = tf32_hi(vv[1]);
      hi.z = tf32_hi(vv[2]);
      hi.w = tf32_hi(vv[3]);
      lo.x = vv[0] - hi.x;
      lo.y = vv[1] - hi.y;
      lo.z = vv[2] - hi.z;
      lo.w = vv[3] - hi.w;
      *(float4*)((unsigned char*)Ahi + off) = hi;
      *(float4*)((unsigned char*)Alo + off) = lo;
    }
    // make the generic-proxy shared-memory writes visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;\n" ::);
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const uint32_t idesc = make_idesc(N);
      const uint32_t a_lbo = kTM * 16, b_lbo = (uint32_t)N * 16;
      const float* As[3] = {Ahi, Ahi, Alo};
      const float* Bs[3] = {Bhi, Blo, Bhi};
      int first = 1;
      for (int pass = 0; pass < 3; ++pass)
        for (int s = 0; s < K / 8; ++s) {
          const uint64_t ad = make_desc(smem_u32(As[pass]) + (uint32_t)(2 * s) * a_lbo, a_lbo, 128);
          const uint64_t bd = make_desc(smem_u32(Bs[pass]) + (uint32_t)(2 * s) * b_lbo, b_lbo, 128);
          const uint32_t acc = first ? 0u : 1u;
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
          first = 0;
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(mbar)));
    }
    // wait for the accumulator
    {
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(mbar)), "r"(phase));
      }
      phase ^= 1u;
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    // epilogue: warp w reads TMEM lanes [32 (w%4), +32) (= tile rows) and the column slice w/4; 8 fp32 columns per
    // tcgen05.ld into a padded shared tile, then every warp writes whole rows with coalesced float2 stores
    {
      const int q4 = warp & 3, slice = warp >> 2, nsl = kTCThreads / 128;
      const int i = q4 * 32 + lane;
      const int DP = NMAX + 1;
      for (int ch = slice; ch < N / 8; ch += nsl) {
        const int c0 = ch * 8;
        uint32_t r[8];
        const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
#pragma unroll
        for (int q = 0; q < 8; ++q) Dst[i * DP + c0 + q] = __uint_as_float(r[q]);
      }
      __syncthreads();
      for (int ii = warp; ii < kTM; ii += kTCThreads / 32) {
        const int64_t row = tm.row0 + ii;
        if (row >= rows_l) break;
        const int64_t p = row / (l + 1);
        const int m = (int)(row - p * (l + 1));
        float2* out = M + p * half_size(L) + half_offset(l) + (int64_t)m * w;
        for (int q = lane; q < w; q += 32) out[q] = make_float2(Dst[ii * DP + 2 * q], Dst[ii * DP + 2 * q + 1]);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(ncols));
}

}  // namespace

size_t corr_tc_smem_bytes(int L, int R) {
  const int K = 2 * R, NMAX = tile_n(L);
  return sizeof(float) * (size_t)(2 * kTM * K + 2 * NMAX * K + ((kTM * (NMAX + 1) + 3) & ~3)) + 32;
}

bool corr_tc_supported(int L, int R) {
  return tile_n(L) <= 256 && (2 * R) % 8 == 0 && corr_tc_smem_bytes(L, R) <= 220 * 1024;
}

cudaError_t launch_corr_coeffs_tc(const float2* F, const float2* H, int64_t B, int L, int Lmax, int R, float2* M,
                                  int num_sms, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  int64_t ntiles = 0;
  for (int l = 0; l <= L; ++l) ntiles += (B * (l + 1) + kTM - 1) / kTM;
  const size_t bytes = corr_tc_smem_bytes(L, R);
  cudaError_t e = cudaFuncSetAttribute(k_corr_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(ntiles, num_sms);
  k_corr_tc<<<grid, kTCThreads, bytes, s>>>(F, H, B, L, Lmax, R, ntiles, M);
  return cudaGetLastError();
}

}  // namespace matcha
