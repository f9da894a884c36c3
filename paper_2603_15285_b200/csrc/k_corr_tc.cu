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
// on an mbarrier; the warps read the 128 x N fp32 accumulator out of TMEM with tcgen05.ld (one TMEM lane per
// row) and store the complex rows of M straight from registers.  A and the accumulator are double-buffered, so
// staging tile t+1 and draining tile t-1 overlap the MMAs of tile t.  Persistent CTAs walk contiguous tile
// ranges l-major, so B is rebuilt only when l changes.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace matcha {

namespace {

constexpr int kTM = 128;          // UMMA_M (rows per tile, one TMEM lane per row)
constexpr int kTCThreads = 512;   // 16 warps: warp w reads TMEM lane quarter w % 4, column slice w / 4
constexpr int kStageUnroll = 4;   // 16-byte A loads in flight per thread
constexpr int kMaxChunks = 8;     // 8-column TMEM chunks per warp in the epilogue (4 slices x 8 x 8 = 256 columns)

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

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase));
  }
}

// Warp-specialised two-deep pipeline per CTA: 16 worker warps stage tile t (B when l changes, A = the tile's F rows
// split into tf32 hi/lo) into A buffer t & 1 and hand it to the MMA warp through an mbarrier; the MMA warp issues the
// 3 x (2R/8) MMAs into accumulator t & 1 and commits; meanwhile the workers drain tile t - 1 from the other
// accumulator straight to global memory.
// RC: compile-time shell count (0 = runtime), so the staging index arithmetic reduces to shifts
template <int RC>
__global__ void __launch_bounds__(kTCThreads + 32, 1)
    k_corr_tc(const float2* __restrict__ F, const float2* __restrict__ H, int64_t B, int L, int Lmax, int Rr,
              int64_t ntiles, float2* __restrict__ M, int dbg) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int R = RC ? RC : Rr;
  const int K = 2 * R;                       // real K (multiple of 8: R % 4 == 0)
  const int NMAX = tile_n(L);
  // layout: A_hi, A_lo [2 buffers][128 x K], B_hi, B_lo [NMAX x K] (fp32 words), row tables, mbarriers, tmem slot
  float* Abuf = (float*)smem;                // buffer b: hi at Abuf + 2b*128K, lo at + (2b+1)*128K
  float* Bhi = Abuf + 4 * kTM * K;
  float* Blo = Bhi + NMAX * K;
  int64_t* rowF = (int64_t*)(Blo + NMAX * K);  // [2][128] F offset of the tile row (complex units), -1 = padding
  int64_t* rowM = rowF + 2 * kTM;              // [2][128] M offset of the tile row
  uint64_t* full = (uint64_t*)(rowM + 2 * kTM);  // [2] A[buf] staged (512 arrivals)
  uint64_t* done = full + 2;                     // [2] MMAs of A[buf] complete
  uint32_t* tslot = (uint32_t*)(done + 2);
  int* cmd = (int*)(tslot + 1);                  // [2] N of the tile in A[buf] (0 = exit)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncf = ncoef(Lmax);
  const uint32_t cols1 = (uint32_t)tmem_cols(NMAX), ncols = 2 * cols1;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&full[b])), "r"(kTCThreads));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&done[b])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tslot;

  if (warp == kTCThreads / 32) {
    // ================================================================ MMA warp
    if (lane == 0) {
      uint32_t fph = 0u;
      const uint32_t a_lbo = kTM * 16;
      for (uint32_t it = 0;; ++it) {
        const int buf = (int)(it & 1);
        mbar_wait(smem_u32(&full[buf]), (fph >> buf) & 1u);
        fph ^= 1u << buf;
        const int N = cmd[buf];
        if (N == 0) break;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        if (dbg & 1) {
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&done[buf])));
          continue;
        }
        const uint32_t idesc = make_idesc(N);
        const uint32_t b_lbo = (uint32_t)N * 16;
        const float* Ahi = Abuf + (2 * buf) * kTM * K;
        const float* Alo = Ahi + kTM * K;
        const uint32_t dt = tmem + (uint32_t)buf * cols1;
        const uint64_t astep = (uint64_t)((2 * a_lbo) >> 4), bstep = (uint64_t)((2 * b_lbo) >> 4);
        for (int pass = 0; pass < 3; ++pass) {
          uint64_t ad = make_desc(smem_u32(pass == 2 ? Alo : Ahi), a_lbo, 128);
          uint64_t bd = make_desc(smem_u32(pass == 1 ? Blo : Bhi), b_lbo, 128);
          for (int s = 0; s < K / 8; ++s) {
            const uint32_t acc = (pass | s) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            ad += astep;
            bd += bstep;
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&done[buf])));
      }
    }
    __syncwarp();
  } else {
    // ================================================================ worker warps
    auto wbar = []() { asm volatile("bar.sync 1, %0;\n" ::"r"(kTCThreads)); };
    uint32_t dph = 0u;  // bit b: parity of the next completion of done[b]
    int cur_l = -1;
    // contiguous tile ranges per CTA (tiles enumerated l-major: degree l has ceil(B (l+1) / 128) tiles), so B is
    // rebuilt about once per CTA; the (l, first row) of the range start is found once, then advanced incrementally
    const int64_t t_begin = ntiles * blockIdx.x / gridDim.x, t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
    int l = 0;
    int64_t row0 = 0;
    {
      int64_t t = t_begin;
      for (l = 0; l <= L; ++l) {
        const int64_t nt = (B * (l + 1) + kTM - 1) / kTM;
        if (t < nt) break;
        t -= nt;
      }
      row0 = t * kTM;
    }
    int prev_l = -1, prev_n = 0;
    for (int64_t t = t_begin; t <= t_end; ++t) {
      const int buf = (int)((t - t_begin) & 1);
      const bool have = t < t_end;
      const int w = 2 * l + 1, N = tile_n(l);
      wbar();  // row tables / A[buf] of tile t - 2 are no longer read (its drain finished in the last iteration)
      if (have) {
        const int64_t rows_l = B * (l + 1);
        if (l != cur_l) {
          // B operand for degree l: the tensor core must be done with the old one (tile t - 1)
          if (t > t_begin) mbar_wait(smem_u32(&done[buf ^ 1]), (dph >> (buf ^ 1)) & 1u);
          const float2* Hl = H + (int64_t)lm_index(l, 0) * R;
          for (int e = tid; e < (N / 2) * R; e += kTCThreads) {
            const int nn = e / R, r = e - nn * R;  // output complex column nn (padded to N/2)
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
            const float v[4] = {hre, -him, him, hre};
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
          cur_l = l;
        }
        // row tables of this tile: (p, m) -> F row and M row offsets
        for (int i = tid; i < kTM; i += kTCThreads) {
          const int64_t row = row0 + i;
          int64_t fo = -1, mo = -1;
          if (row < rows_l) {
            const int64_t pp = row / (l + 1);
            const int m = (int)(row - pp * (l + 1));
            fo = (pp * ncf + lm_index(l, m)) * R;
            mo = pp * half_size(L) + half_offset(l) + (int64_t)m * w;
          }
          rowF[buf * kTM + i] = fo;
          rowM[buf * kTM + i] = mo;
        }
        wbar();
        // A operand: 128 rows (p, m) of F, interleaved complex along k, split into tf32 hi + lo; all of a thread's
        // 16-byte loads are issued before any is consumed
        float* Ahi = Abuf + (2 * buf) * kTM * K;
        float* Alo = Ahi + kTM * K;
        const int k4n = K / 4, nel = kTM * k4n;
        for (int e0 = 0; e0 < nel; e0 += kStageUnroll * kTCThreads) {
          float4 v[kStageUnroll];
#pragma unroll
          for (int u = 0; u < kStageUnroll; ++u) {
            const int e = e0 + u * kTCThreads + tid;
            v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (e < nel) {
              const int i = e / k4n, k4 = e - i * k4n;
              const int64_t fo = rowF[buf * kTM + i];
              if (fo >= 0 && !(dbg & 2)) v[u] = __ldg(reinterpret_cast<const float4*>(F + fo) + k4);
            }
          }
#pragma unroll
          for (int u = 0; u < kStageUnroll; ++u) {
            const int e = e0 + u * kTCThreads + tid;
            if (e >= nel) break;
            const int i = e / k4n, k4 = e - i * k4n;
            const uint32_t off = kmaj_off(i, 4 * k4, kTM);  // 4 consecutive k = one 16-byte chunk
            float4 hi, lo;
            hi.x = tf32_hi(v[u].x);
            hi.y = tf32_hi(v[u].y);
            hi.z = tf32_hi(v[u].z);
            hi.w = tf32_hi(v[u].w);
            lo.x = v[u].x - hi.x;
            lo.y = v[u].y - hi.y;
            lo.z = v[u].z - hi.z;
            lo.w = v[u].w - hi.w;
            *(float4*)((unsigned char*)Ahi + off) = hi;
            *(float4*)((unsigned char*)Alo + off) = lo;
          }
        }
        // hand A[buf] (and B) to the MMA warp
        if (tid == 0) cmd[buf] = N;
        asm volatile("fence.proxy.async.shared::cta;\n" ::);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&full[buf])) : "memory");
      }
      // drain tile t - 1 (overlaps the MMAs of tile t): warp w reads TMEM lane quarter w % 4 (= tile rows) and a
      // contiguous range of 8-column chunks; all tcgen05.ld of the range are issued before one wait
      if (t > t_begin) {
        const int pb = buf ^ 1;
        mbar_wait(smem_u32(&done[pb]), (dph >> pb) & 1u);
        dph ^= 1u << pb;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const int q4 = warp & 3, slice = warp >> 2, nsl = kTCThreads / 128;
        const int pw = 2 * prev_l + 1, nch = prev_n / 8;
        const int ch0 = nch * slice / nsl, ch1 = nch * (slice + 1) / nsl;
        // tcgen05.ld.16x256b: thread t receives rows (t / 4, t / 4 + 8) of the 16-lane half, columns 2 (t % 4) and
        // 2 (t % 4) + 1 of the 8-column chunk = one complex value per row; four consecutive threads cover 32
        // contiguous bytes of an M row, so every store instruction writes 8 full sectors
        const int t4 = lane & 3, trow = lane >> 2;
        int64_t mrow[4];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          mrow[2 * hh] = rowM[pb * kTM + q4 * 32 + 16 * hh + trow];
          mrow[2 * hh + 1] = rowM[pb * kTM + q4 * 32 + 16 * hh + 8 + trow];
        }
        for (int cb = ch0; cb < ch1; cb += 4) {  // four 8-column chunks per wait
          uint32_t r[4][2][4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (cb + u < ch1)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh)
                asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];\n"
                             : "=r"(r[u][hh][0]), "=r"(r[u][hh][1]), "=r"(r[u][hh][2]), "=r"(r[u][hh][3])
                             : "r"(tmem + (uint32_t)pb * cols1 + ((uint32_t)(q4 * 32 + 16 * hh) << 16) +
                                   (uint32_t)(8 * (cb + u))));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
          if (!(dbg & 4)) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int cc = 4 * (cb + u) + t4;  // complex column
              if (cb + u < ch1 && cc < pw)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                  if (mrow[2 * hh] >= 0)
                    M[mrow[2 * hh] + cc] = make_float2(__uint_as_float(r[u][hh][0]), __uint_as_float(r[u][hh][1]));
                  if (mrow[2 * hh + 1] >= 0)
                    M[mrow[2 * hh + 1] + cc] = make_float2(__uint_as_float(r[u][hh][2]), __uint_as_float(r[u][hh][3]));
                }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      }
      if (have) {
        prev_l = l;
        prev_n = N;
        row0 += kTM;
        if (row0 >= B * (l + 1)) {
          ++l;
          row0 = 0;
        }
      }
    }
    // stop the MMA warp
    const int fb = (int)((t_end - t_begin) & 1);
    if (tid == 0) cmd[fb] = 0;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&full[fb])) : "memory");
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(ncols));
}

}  // namespace

size_t corr_tc_smem_bytes(int L, int R) {
  const int K = 2 * R, NMAX = tile_n(L);
  return sizeof(float) * (size_t)(4 * kTM * K + 2 * NMAX * K) + sizeof(int64_t) * 4 * kTM + 64;
}

bool corr_tc_supported(int L, int R) {
  return 2 * tmem_cols(tile_n(L)) <= 512 && (2 * R) % 8 == 0 && corr_tc_smem_bytes(L, R) <= 220 * 1024;
}

cudaError_t launch_corr_coeffs_tc(const float2* F, const float2* H, int64_t B, int L, int Lmax, int R, float2* M,
                                  int num_sms, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  int64_t ntiles = 0;
  for (int l = 0; l <= L; ++l) ntiles += (B * (l + 1) + kTM - 1) / kTM;
  const size_t bytes = corr_tc_smem_bytes(L, R);
  auto kern = R == 32 ? k_corr_tc<32> : R == 16 ? k_corr_tc<16> : k_corr_tc<0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(ntiles, num_sms);
  const char* dv = getenv("MATCHA_CORR_DBG");
  kern<<<grid, kTCThreads + 32, bytes, s>>>(F, H, B, L, Lmax, R, ntiles, M, dv ? atoi(dv) : 0);
  return cudaGetLastError();
}

}  // namespace matcha
