// k_sh_tc.cu -- stage 1 (shell SH analysis), ring sampling + ring DFT with the DFT on the 5th-generation tensor
// cores (tcgen05.mma kind::f16, fp16 hi/lo split, A operand in TMEM), FP32 handles.
//
// north_star stage (1); readings C2-C5:
//   G_ijm = (2 pi / n_phi) sum_k u(c + t + r_i w_jk) e^{-i m phi_k}     (ring (i, j): shell r_i, polar node theta_j)
// followed by the Legendre contraction f_lm(r_i) = sum_j W_j Pbar_lm(x_j) G_ijm (k_sh_legendre_pers in k_sh.cu).
//
// The ring DFT is a dense real contraction  D[o][ring] = sum_k A[o][k] S[ring][k]  with o = 2m + (0: Re, 1: Im),
// A[2m][k] = (2 pi / n_phi) cos(m phi_k), A[2m+1][k] = -(2 pi / n_phi) sin(m phi_k), S = the ring samples (folded
// over the real-data symmetry to Kh + 1 k-columns per parity class).  It runs as tcgen05.mma with M = 128 DFT rows
// (2(L+1) <= 128 used; at L = 64 the 130th/131st rows, m = 64, are summed by the samplers from the FP32 samples),
// N = 64 rings per tile (one k round per lane, Kh <= 32), 32 or 16 (two rounds, Kh <= 64), K-steps of 16 fp16:
//   A_hi, A_lo  the DFT matrix x 2^10 split into fp16 hi + lo, in TMEM (written once per CTA; constant),
//   S_hi, S_lo  each ring's samples scaled by a power of two and split into fp16 hi + lo, in shared memory
//               (K-major, SWIZZLE_NONE; the K-chunk stride is padded by 16 B so that a warp's consecutive-k stores
//               along one ring hit different banks), double-buffered,
//   D           FP32 accumulator in TMEM (double-buffered), read back with tcgen05.ld: TMEM lane o = output row,
//               column = ring; lane o of a warp stores G[ring][o] (coalesced), undoing the two scales.
//   D = A_hi S_hi + A_hi S_lo + A_lo S_hi  (FP32-level accuracy; lo*lo dropped).
// The MMAs are issued by a dedicated warp (kThr sampler threads + 1 MMA warp), so the ~1.7 k issue cycles per tile
// overlap the sampling of the next tile.
//
// Persistent CTAs (one per SM) take whole particles.  Per particle the rings are sorted by the plane index of their
// z (deterministic counting sort), so consecutive tiles of 64 rings need a small window of z-planes: the planes live
// in a P-slot ring buffer in shared memory, prefetched one tile ahead with cp.async (the particle crosses HBM once);
// 128^3 boxes run with 2 slots (tiles then stay within one z bucket) and the sorted ring list in a global workspace.
// Per tile: sample (trilinear from shared memory) -> S[buf]; the MMA warp issues 3 x K/16 MMAs into D[buf];
// meanwhile the CTA drains D[buf^1] of the previous tile and samples the next one.
// Deterministic: fixed summation orders, no atomics on data.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_fp16.h>

#include "common.cuh"

namespace matcha {

namespace {

constexpr int kThr = 512;
__device__ unsigned long long g_sh_prof[8];  // MATCHA_SH_DBG & 8: cycles per phase, summed over sampler warps
constexpr int kWarps = kThr / 32;
// rings per tile (UMMA_N): 64, or 32 for L > 32 (two k rounds per lane, Kh <= 64: the S buffers of the larger K
// and the bigger planes must fit next to each other)
constexpr int kTM = 128;  // UMMA_M

__host__ __device__ inline int plane_pitch_tc(int N) { return N + 8; }

constexpr int kSlotFields = 2;  // per ring slot: G offset, 1/(1024 scale) (read by the drain one tile later)

struct TcLayout {
  size_t tw, node, planes, B, list, slots, tiles, misc, total;
  int Kp, Kc, lbo, P, maxtiles;
};

// glist: the z-sorted ring list lives in a global workspace instead of shared memory (large boxes)
__host__ __device__ inline TcLayout tc_layout(int N, int R, int nth, int nph, int P, int NR, bool glist = false) {
  TcLayout s;
  s.Kp = (nph + 15) / 16 * 16;  // K padded to the fp16 MMA K-step
  s.Kc = s.Kp / 8;              // 16-byte K chunks (8 fp16)
  s.lbo = NR * 16 + 16;         // K-chunk stride, padded by 16 B against bank conflicts
  s.P = P;
  s.maxtiles = (R * nth + NR - 1) / NR + N + 4;
  size_t o = 0;
  auto take = [&](size_t b, size_t al) {
    o = (o + al - 1) / al * al;
    size_t r = o;
    o += b;
    return r;
  };
  s.B = take((size_t)4 * s.Kc * s.lbo, 1024);  // [buf][hi, lo][Kc][lbo]
  s.tw = take(sizeof(float2) * nph, 16);
  s.node = take(sizeof(float2) * nth, 16);
  s.planes = take(sizeof(float) * (size_t)P * N * plane_pitch_tc(N), 16);
  s.list = take(glist ? 0 : sizeof(int) * (size_t)R * nth, 16);
  s.slots = take(sizeof(int) * 3 * kSlotFields * NR, 16);
  s.tiles = take(sizeof(int) * ((size_t)3 * s.maxtiles + 1 + (N + 4) + (N + 2)), 16);
  s.misc = take(64 + sizeof(int) * (4 + kWarps), 16);
  s.total = o;
  return s;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_nosw(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // sm_100 descriptor version
  return d;
}

__host__ __device__ inline uint32_t idesc_f16(int M, int N) {
  uint32_t d = 0;
  d |= 1u << 4;                   // D = F32; A = B = F16 (format 0), both K-major
  d |= (uint32_t)(N >> 3) << 17;  // n_dim
  d |= (uint32_t)(M >> 4) << 24;  // m_dim
  return d;
}

__host__ __device__ inline uint32_t idesc_tf32(int M, int N) {
  uint32_t d = 0;
  d |= 1u << 4;                   // D = F32
  d |= 2u << 7;                   // A = TF32
  d |= 2u << 10;                  // B = TF32
  d |= (uint32_t)(N >> 3) << 17;  // n_dim
  d |= (uint32_t)(M >> 4) << 24;  // m_dim
  return d;
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, bool valid) {
  const unsigned s = su32(sdst);
  const int n = valid ? 16 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(n));
}

// the particle volumes are read exactly once: mark their L2 lines evict-first so that the ring coefficients G
// (written here, read back by the Legendre kernel) stay in L2 instead of round-tripping through HBM
__device__ __forceinline__ void cp_async16_stream(void* sdst, const void* gsrc, bool valid, uint64_t policy) {
  const unsigned s = su32(sdst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(s), "l"(gsrc), "r"(n),
               "l"(policy));
}

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

// same, but the waiting thread is suspended in hardware between checks (for the otherwise idle MMA warp, so that
// it does not take issue slots from the sampler warps)
__device__ __forceinline__ void mbar_wait_suspend(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase), "r"(1000000u));
  }
}

// trilinear sample from the plane ring buffer: b0 = plane of floor(z) at (0, 0), dz = offset (floats) of plane
// floor(z)+1 relative to it; both planes are resident (zero planes outside the volume), so only x, y are tested.
template <int NT>
__device__ __forceinline__ float tri_xy(const float* __restrict__ b0, int dz, int Nr, float px, float py, float fz) {
  const int N = NT ? NT : Nr;
  const int W = plane_pitch_tc(N);
  const float fx0 = floorf(px), fy0 = floorf(py);
  const int x0 = (int)fx0, y0 = (int)fy0;
  const float fx = px - fx0, fy = py - fy0;
  float c[8];
  if ((unsigned)x0 < (unsigned)(N - 1) && (unsigned)y0 < (unsigned)(N - 1)) {
    const float* b = b0 + y0 * W + x0;
    c[0] = b[0];
    c[1] = b[1];
    c[2] = b[W];
    c[3] = b[W + 1];
    c[4] = b[dz];
    c[5] = b[dz + 1];
    c[6] = b[dz + W];
    c[7] = b[dz + W + 1];
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int x = x0 + (q & 1), y = y0 + ((q >> 1) & 1);
      const bool in = x >= 0 && y >= 0 && x < N && y < N;
      c[q] = in ? b0[((q >> 2) ? dz : 0) + y * W + x] : 0.f;
    }
  }
  const float c00 = fmaf(fx, c[1] - c[0], c[0]);
  const float c01 = fmaf(fx, c[3] - c[2], c[2]);
  const float c10 = fmaf(fx, c[5] - c[4], c[4]);
  const float c11 = fmaf(fx, c[7] - c[6], c[6]);
  const float c0 = fmaf(fy, c01 - c00, c00);
  const float c1 = fmaf(fy, c11 - c10, c10);
  return fmaf(fz, c1 - c0, c0);
}

// four samples of one ring (mirrored phi indices) with one x/y bounds test, loads issued back to back
template <int NT>
__device__ __forceinline__ void tri4_xy(const float* __restrict__ b0, int dz, int Nr, const float* px, const float* py,
                                        float fz, float* out) {
  const int N = NT ? NT : Nr;
  const int W = plane_pitch_tc(N);
  int x0[4], y0[4];
  float fx[4], fy[4];
  bool ok = true;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float fx0 = floorf(px[q]), fy0 = floorf(py[q]);
    x0[q] = (int)fx0;
    y0[q] = (int)fy0;
    fx[q] = px[q] - fx0;
    fy[q] = py[q] - fy0;
    ok = ok && (unsigned)x0[q] < (unsigned)(N - 1) && (unsigned)y0[q] < (unsigned)(N - 1);
  }
  if (ok) {
    float c[4][8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float* b = b0 + y0[q] * W + x0[q];
      c[q][0] = b[0];
      c[q][1] = b[1];
      c[q][2] = b[W];
      c[q][3] = b[W + 1];
      c[q][4] = b[dz];
      c[q][5] = b[dz + 1];
      c[q][6] = b[dz + W];
      c[q][7] = b[dz + W + 1];
    }
    // the seven lerps of two samples at a time on the packed FP32x2 pipe (FFMA2): lerp(a, b, f) = f b + (1 - f) a
    // as fma(f, b, fma(-f, a, a))
    const float2 fz2 = make_float2(fz, fz), nfz2 = make_float2(-fz, -fz);
    auto lerp2 = [](float2 a, float2 b, float2 f, float2 nf) { return __ffma2_rn(f, b, __ffma2_rn(nf, a, a)); };
#pragma unroll
    for (int pq = 0; pq < 4; pq += 2) {
      float2 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = make_float2(c[pq][k], c[pq + 1][k]);
      const float2 fx2 = make_float2(fx[pq], fx[pq + 1]), nfx2 = make_float2(-fx[pq], -fx[pq + 1]);
      const float2 fy2 = make_float2(fy[pq], fy[pq + 1]), nfy2 = make_float2(-fy[pq], -fy[pq + 1]);
      const float2 c00 = lerp2(v[0], v[1], fx2, nfx2), c01 = lerp2(v[2], v[3], fx2, nfx2);
      const float2 c10 = lerp2(v[4], v[5], fx2, nfx2), c11 = lerp2(v[6], v[7], fx2, nfx2);
      const float2 c0 = lerp2(c00, c01, fy2, nfy2), c1 = lerp2(c10, c11, fy2, nfy2);
      const float2 o = lerp2(c0, c1, fz2, nfz2);
      out[pq] = o.x;
      out[pq + 1] = o.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = tri_xy<NT>(b0, dz, N, px[q], py[q], fz);
  }
}

// K order of the ring samples: position 4(k-1)+q (k = 1..Kh, q = 0..3) holds phi index {k, k+Mp, Mp-k, 2Mp-k}[q]
// (the four mirrored samples one lane computes, stored with one 8-byte write), then 4 Kh + e holds {0, Mp, Mp/2,
// 3Mp/2}[e]; the DFT matrix A uses the same permutation.
__device__ __forceinline__ int kpos_phi(int c, int Kh, int Mp) {
  if (c < 4 * Kh) {
    const int k = c / 4 + 1, q = c & 3;
    return q == 0 ? k : q == 1 ? k + Mp : q == 2 ? Mp - k : 2 * Mp - k;
  }
  const int e = c - 4 * Kh;
  return e == 0 ? 0 : e == 1 ? Mp : e == 2 ? Mp / 2 : 3 * Mp / 2;
}

__device__ __forceinline__ uint32_t pack_h2(float lo16, float hi16) {
  const __half2 h = __floats2half2_rn(lo16, hi16);  // .x = first (low 16 bits) = even k
  return *reinterpret_cast<const uint32_t*>(&h);
}

// NR rings per tile, KR rounds of 32 k per lane (Kh <= 32 KR)
template <int NT, int NR, int KR>
__global__ void __launch_bounds__(kThr + 32, 1)
    k_sh_rings_tc(const float* __restrict__ vols, int64_t B, const float* __restrict__ shifts, int shift_stride,
                  ShTables<float> tab, int P, float2* __restrict__ G, int* __restrict__ flags, int dbg) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int N = NT ? NT : tab.N;
  const int R = tab.R, L = tab.L, nth = tab.nth, nph = tab.nph;
  const int Mp = nph / 2, Kh = (Mp - 1) / 2;
  const bool mid = (Mp % 2) == 0;
  const TcLayout lay = tc_layout(N, R, nth, nph, P, NR, tab.tc_list != nullptr);
  const int Kp = lay.Kp, Kc = lay.Kc, LBO = lay.lbo;
  const int PW = plane_pitch_tc(N), PS = N * PW;
  unsigned char* Bs = smem + lay.B;  // buffer b: hi at Bs + (2b) Kc LBO, lo at + (2b+1) Kc LBO
  float2* tw = (float2*)(smem + lay.tw);
  float2* node = (float2*)(smem + lay.node);
  float* planes = (float*)(smem + lay.planes);
  int* list = tab.tc_list ? tab.tc_list + (size_t)blockIdx.x * R * nth : (int*)(smem + lay.list);
  int* cnt = (int*)(smem + lay.planes);  // counting-sort table [N+3][nth], aliases the planes between particles
  int* slots = (int*)(smem + lay.slots);  // [3 tiles][kSlotFields][NR]
  int* tstart = (int*)(smem + lay.tiles);  // [max tiles + 1] first ring of each tile
  int* tlo = tstart + lay.maxtiles + 1;     // [max tiles] lowest plane
  int* thi = tlo + lay.maxtiles;            // [max tiles] highest plane
  int* boff = thi + lay.maxtiles;           // [N+4] first ring of each z bucket
  int* zslot = boff + (N + 4);              // [N+2] plane slot of z = -1 .. N
  uint64_t* full = (uint64_t*)(smem + lay.misc);  // [2] S[buf] written (512 arrivals)
  uint64_t* done = full + 2;                      // [2] MMAs of S[buf] complete (tcgen05.commit)
  uint32_t* tslot = (uint32_t*)(done + 2);
  int* cmd = (int*)(tslot + 1);   // [2] 1 = run the MMAs of this buffer, 0 = exit
  int* s_nt = cmd + 2;            // tiles of the current particle
  int* s_wtot = s_nt + 1;         // [kWarps] scan scratch
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nrow = 2 * (L + 1);
  const float dscale = (float)(2.0 * kPi) / (float)nph;
  const int nrings = R * nth;
  const int nbk = N + 3;  // z buckets: clamp(floor z, -2, N) + 2

  // ---- one-time setup: tables, TMEM, mbarriers, A (DFT matrix x 2^10, fp16 hi/lo) in TMEM, zero K padding
  for (int t = tid; t < nph; t += blockDim.x) tw[t] = tab.tw[t];
  for (int t = tid; t < nth; t += blockDim.x) node[t] = tab.node[t];
  for (int t = tid; t < N + 2; t += blockDim.x) zslot[t] = (t - 1 + P) % P;
  for (int t = tid; t < 4 * Kc * (LBO / 16); t += blockDim.x) {
    const int chunk = (t / (LBO / 16)) % Kc;  // 8 fp16 k per chunk; zero the chunks holding padding k >= nph
    if (8 * chunk + 7 >= nph) reinterpret_cast<float4*>(Bs)[t] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&full[b])), "r"(kThr));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&done[b])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tslot;
  const uint32_t colA_hi = 0, colA_lo = (uint32_t)(Kp / 2);  // 2 fp16 per 32-bit TMEM column
  const uint32_t colD = (uint32_t)((Kp + 31) / 32 * 32);
  if (warp < kWarps) {
    const int q = warp & 3, g = warp >> 2;
    const int o = 32 * q + lane, m = o >> 1;
    for (int ch = g; ch < Kp / 16; ch += 4) {  // 16 k = 8 columns per tcgen05.st
      uint32_t hi[8], lo[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float v2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 16 * ch + 2 * u + h;  // K position -> phi index (see the sampler's K order)
          const int kphi = kpos_phi(c, Kh, Mp);
          float v = 0.f;
          if (o < nrow && c < nph) {
            const float2 e = tw[(int)(((long long)m * kphi) % nph)];
            v = ((o & 1) ? -e.y : e.x) * dscale * 1024.f;
          }
          v2[h] = v;
        }
        const float h0 = __half2float(__float2half_rn(v2[0])), h1 = __half2float(__float2half_rn(v2[1]));
        hi[u] = pack_h2(v2[0], v2[1]);
        lo[u] = pack_h2(v2[0] - h0, v2[1] - h1);
      }
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(
                       ta + colA_hi + 8 * ch),
                   "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3]), "r"(hi[4]), "r"(hi[5]), "r"(hi[6]), "r"(hi[7]));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(
                       ta + colA_lo + 8 * ch),
                   "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();

  // ================================================================ MMA warp
  if (warp == kWarps) {
    if (lane == 0 && !(dbg & 1)) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const uint32_t idesc = idesc_f16(kTM, NR);
      const uint64_t step = (uint64_t)((2 * LBO) >> 4);  // one K-step (16 fp16) = two 16-byte core-matrix columns
      uint32_t fph = 0u;
      for (uint32_t it = 0;; ++it) {
        const int buf = (int)(it & 1);
        mbar_wait_suspend(su32(&full[buf]), (fph >> buf) & 1u);
        fph ^= 1u << buf;
        if (!cmd[buf]) break;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const unsigned char* Shi = Bs + (size_t)(2 * buf) * Kc * LBO;
        const uint64_t dhi = desc_nosw(su32(Shi), LBO, 128), dlo = desc_nosw(su32(Shi + (size_t)Kc * LBO), LBO, 128);
        const uint32_t dcol = tmem + colD + (uint32_t)(NR * buf);
        for (int pass = 0; pass < 3; ++pass) {
          uint32_t acol = tmem + (pass == 2 ? colA_lo : colA_hi);
          uint64_t bd = (pass == 1) ? dlo : dhi;
          for (int s = 0; s < Kp / 16; ++s) {
            const uint32_t acc = (pass | s) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(dcol),
                "r"(acol), "l"(bd), "r"(idesc), "r"(acc));
            acol += 8u;
            bd += step;
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            su32(&done[buf])));
      }
    }
    __syncwarp();
  } else {
    // ================================================================ sampler warps (512 threads)
    auto sbar = []() { asm volatile("bar.sync 1, %0;\n" ::"r"(kThr)); };
    auto sbar_or = [](bool v) {  // sampler barrier that also ORs a predicate over the 512 sampler threads
      int r;
      asm volatile(
          "{\n\t.reg .pred p, q;\n\tsetp.ne.s32 q, %1, 0;\n\tbar.red.or.pred p, 1, %2, q;\n\tselp.s32 %0, 1, 0, p;\n\t}\n"
          : "=r"(r)
          : "r"((int)v), "n"(kThr));
      return r != 0;
    };
    uint32_t dph = 0u;       // bit b: parity of the next completion of done[b]
    uint64_t l2_stream;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(l2_stream));
    uint32_t gtile = 0;      // global tile counter (buffer = gtile & 1)
    // this lane's ring positions (the same for every ring): phi indices k, k + Mp, Mp - k, 2Mp - k per k round, and
    // the extra sample xe (phi index 0, Mp, Mp/2, 3Mp/2) of the warp's ring xr
    const int nx = mid ? 4 : 2;
    float2 ph[KR][4];
    auto load_ph = [&]() {
#pragma unroll
      for (int kr = 0; kr < KR; ++kr) {
        const int k = 32 * kr + lane + 1;  // Kh <= 32 KR (host-checked)
        const int kk[4] = {k, k + Mp, Mp - k, 2 * Mp - k};
#pragma unroll
        for (int q = 0; q < 4; ++q) ph[kr][q] = tw[k <= Kh ? kk[q] : 0];
      }
    };
    load_ph();
    const int xr = lane / nx, xe = lane % nx;
    const int xcol = xe == 0 ? 0 : xe == 1 ? Mp : xe == 2 ? Mp / 2 : 3 * Mp / 2;
    for (int64_t p = blockIdx.x; p < B; p += gridDim.x) {
      const float* vol = vols + p * (int64_t)N * N * N;
      const float cc = 0.5f * (float)(N - 1);
      float cx = cc, cy = cc, cz = cc;
      if (shifts) {
        cx += shifts[p * shift_stride + 0];
        cy += shifts[p * shift_stride + 1];
        cz += shifts[p * shift_stride + 2];
      }
      auto zfloor = [&](int i, int j) -> int { return (int)floorf(fmaf((float)i + 0.5f, node[j].x, cz)); };
      auto bucket = [&](int zb) { return min(max(zb, -2), N) + 2; };

      long long tp0 = (dbg & 8) ? clock64() : 0;
      // ---- 1. counting sort of the rings by z bucket, then (j, i), one item per ring.  For fixed j the bucket is
      //      monotone in i, so the rings of cell (bucket, j) are a contiguous i-range whose first i gives each ring
      //      its rank: deterministic without ordered atomics.
      int* cstart = cnt + nbk * nth;  // first i of each (bucket, j) cell (also aliases the planes)
      for (int t = tid; t < nbk * nth; t += kThr) cnt[t] = 0;
      sbar();
      for (int e = tid; e < nrings; e += kThr) {
        const int j = e / R, i = e - j * R;
        const int b = bucket(zfloor(i, j));
        atomicAdd(&cnt[b * nth + j], 1);
        if (i == 0 || bucket(zfloor(i - 1, j)) != b) cstart[b * nth + j] = i;
      }
      sbar();
      {
        const int E = nbk * nth, per = (E + kThr - 1) / kThr;
        const int e0 = min(E, tid * per), e1 = min(E, e0 + per);
        int sum = 0;
        for (int e = e0; e < e1; ++e) sum += cnt[e];
        int v = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += u;
        }
        if (lane == 31) s_wtot[warp] = v;
        sbar();
        int off = 0;
        for (int w = 0; w < warp; ++w) off += s_wtot[w];
        int run = off + v - sum;
        for (int e = e0; e < e1; ++e) {
          const int c = cnt[e];
          cnt[e] = run;
          run += c;
        }
      }
      sbar();
      for (int b = tid; b < nbk; b += kThr) boff[b] = cnt[b * nth];
      if (tid == 0) boff[nbk] = nrings;
      for (int e = tid; e < nrings; e += kThr) {
        const int j = e / R, i = e - j * R;
        const int c = bucket(zfloor(i, j)) * nth + j;
        list[cnt[c] + (i - cstart[c])] = (i << 16) | j;
      }
      sbar();
      if ((dbg & 8) && lane == 0) atomicAdd(&g_sh_prof[0], (unsigned long long)(clock64() - tp0));
      // planes are requested in increasing z; plane z lives in slot zslot[z + 1] = z mod P (it replaces plane z - P,
      // which the current tile no longer needs because every request stays below lo(t) + P).  The first window is
      // requested before the tiles are built (it only depends on the lowest ring), so the load overlaps the build.
      const int zfirst = min(max(bucket(zfloor(list[0] >> 16, list[0] & 0xffff)) - 2, -1), N - 1);
      int zhave = zfirst - 1;
      auto request = [&](int zto) {
        const int n4 = N / 4;
        for (int z = zhave + 1; z <= zto; ++z) {
          float* dst = planes + zslot[z + 1] * PS;
          const bool valid = z >= 0 && z < N;
          const float* src = vol + (size_t)(valid ? z : 0) * N * N;
          if (!(dbg & 16))
            for (int t = tid; t < N * n4; t += kThr) {
              const int y = t / n4, x4 = t - y * n4;
              cp_async16_stream(dst + y * PW + 4 * x4, src + y * N + 4 * x4, valid, l2_stream);
            }
        }
        zhave = max(zhave, zto);
        asm volatile("cp.async.commit_group;\n" ::);
      };
      request(min(zfirst + P - 1, N));
      // ---- 2. tiles: <= NR consecutive rings whose planes fit the P-slot window.  Fixed chunks of NR rings when every
      //      chunk needs <= P planes (the common case: one thread per chunk); otherwise a greedy cut at z-bucket
      //      boundaries by one thread.  The tiling does not change any result (rings are independent MMA columns).
      auto zlo_of = [&](int b) { return min(max(b - 2, -1), N - 1); };
      {
        const int nchunk = (nrings + NR - 1) / NR;
        bool bad = false;
        for (int c = tid; c < nchunk; c += kThr) {
          const int s0 = c * NR, e = min(s0 + NR, nrings);
          const int r0 = list[s0], r1 = list[e - 1];
          const int lo = zlo_of(bucket(zfloor(r0 >> 16, r0 & 0xffff)));
          const int hi = zlo_of(bucket(zfloor(r1 >> 16, r1 & 0xffff))) + 1;
          tstart[c] = s0;
          tlo[c] = lo;
          thi[c] = hi;
          bad = bad || (hi - lo + 1 > P);
        }
        if (tid == 0) {
          tstart[nchunk] = nrings;
          *s_nt = nchunk;
        }
        if (sbar_or(bad) && tid == 0) {
          int nt = 0, s0 = 0;
          while (s0 < nrings) {
            int b0 = 0;
            {
              const int r = list[s0];
              b0 = bucket(zfloor(r >> 16, r & 0xffff));
            }
            const int zl = zlo_of(b0);
            int bx = b0;  // first bucket whose plane is beyond the window
            while (bx < nbk && zlo_of(bx) <= zl + P - 2) ++bx;
            const int e = min(s0 + NR, boff[bx]);
            const int rl = list[e - 1];
            tstart[nt] = s0;
            tlo[nt] = zl;
            thi[nt] = zlo_of(bucket(zfloor(rl >> 16, rl & 0xffff))) + 1;
            ++nt;
            s0 = e;
          }
          tstart[nt] = nrings;
          *s_nt = nt;
        }
      }
      sbar();
      const int ntiles = *s_nt;
      float* const Gp = (float*)(G + p * (int64_t)R * nth * (L + 1));


      for (int t = 0; t <= ntiles; ++t) {
        const uint32_t gcur = gtile;  // global index of tile t (tiles handed to the MMA warp so far)
        const int buf = (int)(gcur & 1);
        long long tq0 = (dbg & 8) ? clock64() : 0;
        if (t < ntiles) {
          // ring geometry of tile t (static per particle: independent of the planes): lane rr < RPW computes ring slot
          // warp + rr * kWarps, then broadcasts.  With one k round it is done before the plane wait, so that its
          // dependent chain overlaps the barrier and the plane wait (measured: -2 % at c2; with two k rounds it stays
          // after the wait: +4 % at 96^3 otherwise, and a runtime choice costs registers everywhere)
          int* sl = slots + (t % 3) * kSlotFields * NR;
          constexpr int RPW = NR / kWarps;  // rings per warp
          float a_rs[RPW], a_fz[RPW], x_rs = 0.f, x_fz = 0.f;
          int a_b0[RPW], a_dz[RPW], a_in[RPW], x_b0 = 0, x_dz = 0, x_in = 0;
          auto geometry = [&]() {
            float g_rs = 0.f, g_fz = 0.f;
            int g_b0 = 0, g_dz = 0, g_in = 0;
            if (lane < RPW) {
              const int r = warp + lane * kWarps, g = tstart[t] + r;
              int goff = -1;
              if (g < tstart[t + 1]) {
                const int ring = list[g];
                const int i = ring >> 16, j = ring & 0xffff;
                const float rad = (float)i + 0.5f;
                const float2 nd = node[j];
                g_rs = rad * nd.y;
                const float z = fmaf(rad, nd.x, cz);
                const float fz0 = floorf(z);
                const int zb = (int)fz0;
                g_fz = z - fz0;
                g_in = (zb >= -1 && zb <= N - 1) && !(dbg & 2);
                if (g_in) {
                  g_b0 = zslot[zb + 1] * PS;
                  g_dz = zslot[zb + 2] * PS - g_b0;
                }
                goff = (i * nth + j) * (L + 1) * 2;
              }
              sl[r] = goff;
            }
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
              a_rs[rr] = __shfl_sync(0xffffffffu, g_rs, rr);
              a_fz[rr] = __shfl_sync(0xffffffffu, g_fz, rr);
              a_b0[rr] = __shfl_sync(0xffffffffu, g_b0, rr);
              a_dz[rr] = __shfl_sync(0xffffffffu, g_dz, rr);
              a_in[rr] = __shfl_sync(0xffffffffu, g_in, rr);
            }
            const int xsrc = min(xr, RPW - 1);
            x_rs = __shfl_sync(0xffffffffu, g_rs, xsrc);
            x_fz = __shfl_sync(0xffffffffu, g_fz, xsrc);
            x_b0 = __shfl_sync(0xffffffffu, g_b0, xsrc);
            x_dz = __shfl_sync(0xffffffffu, g_dz, xsrc);
            x_in = __shfl_sync(0xffffffffu, g_in, xsrc);
          };
          if constexpr (KR == 1) geometry();
          const int lo = tlo[t], hi = thi[t];
          if (hi - lo + 1 > P && tid == 0) atomicOr(flags, FLAG_PLANES);
          if (zhave < hi) {
            // plane z replaces plane z - P in its slot: requesting above tlo[t-1] + P - 1 before every sampler has
            // finished tile t-1 would overwrite a plane that tile may still read, so such planes wait for a barrier
            // (rare with many slots; common with P = 3 at 96^3)
            const int safe = t > 0 ? tlo[t - 1] + P - 1 : INT_MAX;
            if (hi > safe) {
              if (zhave < safe) request(safe);
              sbar();
            }
            request(hi);
          }
          asm volatile("cp.async.wait_group 0;\n" ::);
          sbar();  // planes of tile t resident; all samplers done with iteration t-1 (incl. drain of tile t-2)
          long long tq1 = (dbg & 8) ? clock64() : 0;
          if ((dbg & 8) && lane == 0) atomicAdd(&g_sh_prof[1], (unsigned long long)(tq1 - tq0));
          if (t + 1 < ntiles) {
            const int want = min(thi[t + 1], lo + P - 1);
            if (want > zhave) request(want);
          }
          if ((dbg & 8) && lane == 0) atomicAdd(&g_sh_prof[5], (unsigned long long)(clock64() - tq1));
          if constexpr (KR > 1) geometry();
          // sample tile t into S[buf] (fp16 hi/lo of the per-ring scaled samples): warp w takes ring slots
          // w, w + 16, ...; lanes walk k along the ring (4 mirrored phi indices per lane, one 8-byte store each)
          unsigned char* Shi = Bs + (size_t)(2 * buf) * Kc * LBO;
          unsigned char* Slo = Shi + (size_t)Kc * LBO;
          float sv[KR][RPW][4], ex = 0.f;
#pragma unroll
          for (int rr = 0; rr < RPW; ++rr) {
            const float rs = a_rs[rr], fz = a_fz[rr];
            const int b0 = a_b0[rr], dz = a_dz[rr], in = a_in[rr];
#pragma unroll
            for (int kr = 0; kr < KR; ++kr) {
#pragma unroll
              for (int q = 0; q < 4; ++q) sv[kr][rr][q] = 0.f;
              if (in && 32 * kr + lane + 1 <= Kh) {
                float px[4], py[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  px[q] = fmaf(rs, ph[kr][q].x, cx);
                  py[q] = fmaf(rs, ph[kr][q].y, cy);
                }
                tri4_xy<NT>(planes + b0, dz, N, px, py, fz, sv[kr][rr]);
              }
            }
          }
          // phi indices 0 and Mp (and Mp/2, 3Mp/2 when Mp is even) of the warp's rings: one sample per lane, all
          // rings in one pass
          if (xr < RPW && x_in) {
            const float2 phx = tw[xcol];
            ex = tri_xy<NT>(planes + x_b0, x_dz, N, fmaf(x_rs, phx.x, cx), fmaf(x_rs, phx.y, cy), x_fz);
          }
          // m = L when 2(L+1) = 130 > 128 MMA rows (L = 64): its two DFT rows from the FP32 samples, in the sampler.
          // The lane's mirrored phi indices k, k+Mp, Mp-k, 2Mp-k (n_phi = 2Mp) carry e^{-iL phi} = e, s e, s conj(e),
          // conj(e) with e = e^{-iL phi_k}, s = (-1)^L.
          if (nrow > kTM) {
            const float sgn = (L & 1) ? -1.f : 1.f;
            __syncwarp();  // sl[] written by lane rr above
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
              float re = 0.f, im = 0.f;
#pragma unroll
              for (int kr = 0; kr < KR; ++kr) {
                const int k = 32 * kr + lane + 1;
                if (k <= Kh) {
                  const float2 e = tw[(L * k) % nph];
                  const float* x = sv[kr][rr];
                  re = fmaf(e.x, (x[0] + x[3]) + sgn * (x[1] + x[2]), re);
                  im = fmaf(e.y, (sgn * x[2] + x[3]) - (x[0] + sgn * x[1]), im);
                }
              }
              if (xr == rr) {
                const float2 e = tw[(L * xcol) % nph];
                re = fmaf(ex, e.x, re);
                im = fmaf(-ex, e.y, im);
              }
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) {
                re += __shfl_xor_sync(0xffffffffu, re, o);
                im += __shfl_xor_sync(0xffffffffu, im, o);
              }
              const int goff = sl[warp + rr * kWarps];
              if (lane == 0 && goff >= 0) {
                Gp[goff + 2 * L] = re * dscale;
                Gp[goff + 2 * L + 1] = im * dscale;
              }
            }
          }
          long long tq2 = (dbg & 8) ? clock64() : 0;
          if ((dbg & 8) && lane == 0) atomicAdd(&g_sh_prof[2], (unsigned long long)(tq2 - tq1));
          // per-ring power-of-two scale (max |sample| -> [2^14, 2^15)), fp16 hi/lo split, 8-byte stores
          if (!(dbg & 32)) {
          float mxv[RPW];
#pragma unroll
          for (int rr = 0; rr < RPW; ++rr) {
            mxv[rr] = 0.f;
#pragma unroll
            for (int kr = 0; kr < KR; ++kr)
              mxv[rr] = fmaxf(mxv[rr], fmaxf(fmaxf(fabsf(sv[kr][rr][0]), fabsf(sv[kr][rr][1])),
                                             fmaxf(fabsf(sv[kr][rr][2]), fabsf(sv[kr][rr][3]))));
            if (xr == rr) mxv[rr] = fmaxf(mxv[rr], fabsf(ex));
          }
          // |x| as an unsigned bit pattern orders like the value: one warp-reduce instruction (REDUX) per ring
#pragma unroll
          for (int rr = 0; rr < RPW; ++rr)
            mxv[rr] = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(mxv[rr])));
#pragma unroll
          for (int rr = 0; rr < RPW; ++rr) {
            const int r = warp + rr * kWarps;
            const float mx = mxv[rr];
            const int e = mx > 0.f ? (int)((__float_as_uint(mx) >> 23) & 0xff) - 127 : 0;
            const int es = min(max(14 - e, -100), 100);  // sc = 2^es, 1 / (1024 sc) = 2^-(es + 10)
            const float sc = __uint_as_float((uint32_t)(127 + es) << 23);
            const uint32_t rowoff = (uint32_t)((r >> 3) * 128 + (r & 7) * 16);
#pragma unroll
            for (int kr = 0; kr < KR; ++kr) {
              const int k = 32 * kr + lane + 1;
              if (k <= Kh) {
                const float2 sc2 = make_float2(sc, sc);
                const float2 x01 = __fmul2_rn(make_float2(sv[kr][rr][0], sv[kr][rr][1]), sc2);
                const float2 x23 = __fmul2_rn(make_float2(sv[kr][rr][2], sv[kr][rr][3]), sc2);
                const __half2 h01 = __float22half2_rn(x01), h23 = __float22half2_rn(x23);
                const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
                const __half2 l01 = __float22half2_rn(__fadd2_rn(x01, make_float2(-f01.x, -f01.y)));
                const __half2 l23 = __float22half2_rn(__fadd2_rn(x23, make_float2(-f23.x, -f23.y)));
                const int c = 4 * (k - 1);  // K position of the lane's first sample (8-byte aligned)
                const uint32_t off = (uint32_t)(c >> 3) * LBO + rowoff + (uint32_t)(c & 7) * 2;
                uint2 hv, lv;
                hv.x = *reinterpret_cast<const uint32_t*>(&h01);
                hv.y = *reinterpret_cast<const uint32_t*>(&h23);
                lv.x = *reinterpret_cast<const uint32_t*>(&l01);
                lv.y = *reinterpret_cast<const uint32_t*>(&l23);
                *(uint2*)(Shi + off) = hv;
                *(uint2*)(Slo + off) = lv;
              }
            }
            if (xr == rr) {
              const int c = 4 * Kh + xe;
              const uint32_t off = (uint32_t)(c >> 3) * LBO + rowoff + (uint32_t)(c & 7) * 2;
              const float x = ex * sc;
              const __half h = __float2half_rn(x);
              *(__half*)(Shi + off) = h;
              *(__half*)(Slo + off) = __float2half_rn(x - __half2float(h));
            }
            if (lane == 0) sl[NR + r] = (int)((uint32_t)(127 - es - 10) << 23);
          }
          }
          if ((dbg & 8) && lane == 0) atomicAdd(&g_sh_prof[3], (unsigned long long)(clock64() - tq2));
          // S[buf] -> async proxy; hand the tile to the MMA warp
          cmd[buf] = 1;
          asm volatile("fence.proxy.async.shared::cta;\n" ::);
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&full[buf])) : "memory");
          gtile = gcur + 1;
        }
        long long tq3 = (dbg & 8) ? clock64() : 0;
        // drain tile t - 1 (overlaps the MMAs of tile t): TMEM lane o = output row, 16 ring columns per warp
        if (t > 0 && !(dbg & 1)) {
          const int pb = (int)((gcur - 1) & 1), tp = t - 1;
          const int q = warp & 3, g = warp >> 2;
          mbar_wait(su32(&done[pb]), (dph >> pb) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
          if (32 * q < nrow && 16 * g < NR) {
            uint32_t v[16];
            const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + colD + (uint32_t)(NR * pb + 16 * g);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                           "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                           "=r"(v[14]), "=r"(v[15])
                         : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
            const int o = 32 * q + lane;
            const int* slp = slots + (tp % 3) * kSlotFields * NR + 16 * g;
            if (o < nrow) {
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const int goff = slp[u];
                if (goff >= 0) Gp[goff + o] = __uint_as_float(v[u]) * __int_as_float(slp[NR + u]);
              }
            }
          }
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
        }
        if (t > 0) dph ^= 1u << ((gcur - 1) & 1);
        if ((dbg & 8) && lane == 0) atomicAdd(&g_sh_prof[4], (unsigned long long)(clock64() - tq3));
      }
      sbar();  // the next particle's sort overwrites the list, the slots and the planes
    }
    // stop the MMA warp
    if (tid == 0) cmd[gtile & 1] = 0;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&full[gtile & 1])) : "memory");
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

}  // namespace

// plane slots for the TC ring kernel (0 = not supported for this handle: use the SIMT kernel).  Tiles are cut at
// z-bucket boundaries so that they never need more than P planes; larger P prefetches further ahead.
// Plane slots P and rings per tile NR for a handle (0 = not supported: use the SIMT kernel).  Preferred: 64 rings per
// tile with one k round (Kh <= 32), 32 with two (Kh <= 64), at least 3 plane slots (one tile of prefetch); large
// boxes (128^3: a 128 x 136 plane is 70 KB) fall back to 16-ring tiles and/or 2 plane slots (tiles then stay inside
// one z bucket and each bucket's new plane is loaded between tiles).
int sh_tc_plane_slots(const ShTables<float>& tab, const std::vector<float>& xnode, int* nr_out, int* glist_out) {
  (void)xnode;
  if (2 * (tab.L + 1) > kTM + 2) return 0;  // the MMA's 128 rows hold m < 64; m = L = 64 is computed by the samplers
  const int Mp = tab.nph / 2, Kh = (Mp - 1) / 2;
  if (Kh > 64 || Kh < 1) return 0;  // at most two rounds of 32 k per lane
  if (2 * (tab.L + 1) > kTM && Kh <= 32) return 0;
  const int Kp = (tab.nph + 15) / 16 * 16;
  if (tab.N % 4 || tab.R * tab.nth >= (1 << 22) || tab.nth > 0xffff) return 0;
  const size_t budget = 225 * 1024;
  const int pref = Kh <= 32 ? 64 : 32;
  // {rings per tile, minimum plane slots, ring list in global memory}, in order of preference (measured)
  const int opts[6][3] = {{pref, 3, 0}, {pref, 3, 1}, {16, 3, 0}, {pref, 2, 1}, {16, 2, 0}, {16, 2, 1}};
  for (const auto& o : opts) {
    const int NR = o[0];
    const bool gl = o[2] != 0;
    if (NR == 16 && Kh <= 32) continue;  // 16-ring tiles exist in the two-round variant only
    if ((Kp + 31) / 32 * 32 + 2 * NR > 512) continue;
    int P = o[1];
    if (tc_layout(tab.N, tab.R, tab.nth, tab.nph, P, NR, gl).total > budget) continue;
    while (P < tab.N + 2 && tc_layout(tab.N, tab.R, tab.nth, tab.nph, P + 1, NR, gl).total <= budget) ++P;
    // the counting-sort table aliases the planes
    if ((size_t)2 * (tab.N + 3) * tab.nth * sizeof(int) > (size_t)P * tab.N * plane_pitch_tc(tab.N) * sizeof(float))
      continue;
    *nr_out = NR;
    *glist_out = gl ? 1 : 0;
    return P;
  }
  return 0;
}

cudaError_t launch_sh_rings_tc(const float* vols, int64_t nb, const float* shifts, int shift_stride,
                               const ShTables<float>& tab, int P, float2* G, int* flags, int num_sms,
                               cudaStream_t st) {
  if (nb == 0) return cudaSuccess;
  const int NR = tab.tcNR;
  const size_t bytes = tc_layout(tab.N, tab.R, tab.nth, tab.nph, P, NR, tab.tc_list != nullptr).total;
  const int grid = (int)std::min<int64_t>(nb, num_sms);
  const char* dv = getenv("MATCHA_SH_DBG");  // profiling knob: 1 = no MMA/drain, 2 = no gathers, 16 = no plane loads, 32 = no split/store
  const int dbg = dv ? atoi(dv) : 0;
  cudaError_t e;
  auto go = [&](auto kern) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) kern<<<grid, kThr + 32, bytes, st>>>(vols, nb, shifts, shift_stride, tab, P, G, flags, dbg);
  };
  if (NR == 64) {
    if (tab.N == 32) go(k_sh_rings_tc<32, 64, 1>);
    else if (tab.N == 64) go(k_sh_rings_tc<64, 64, 1>);
    else go(k_sh_rings_tc<0, 64, 1>);
  } else if (NR == 32) {
    if (tab.N == 96) go(k_sh_rings_tc<96, 32, 2>);
    else if (tab.N == 128) go(k_sh_rings_tc<128, 32, 2>);
    else go(k_sh_rings_tc<0, 32, 2>);
  } else {
    if (tab.N == 128) go(k_sh_rings_tc<128, 16, 2>);
    else go(k_sh_rings_tc<0, 16, 2>);
  }
  if (e != cudaSuccess) return e;
  if (dbg & 8) {
    cudaStreamSynchronize(st);
    unsigned long long h[8];
    cudaMemcpyFromSymbol(h, g_sh_prof, sizeof(h));
    fprintf(stderr, "sh_tc prof (warp-cycles, summed): sort %llu  plane-wait %llu  sample %llu (prefetch issue %llu)  "
            "scale+store %llu  drain %llu\n", h[0], h[1], h[2], h[5], h[3], h[4]);
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_sh_prof, z, sizeof(z));
  }
  return cudaGetLastError();
}

}  // namespace matcha
