// mma_probe.cu -- microbenchmark: issue cost / throughput of tcgen05.mma kind::tf32 (M = 128) for several N,
// with A from TMEM (TS) or shared memory (SS), B K-major SWIZZLE_NONE in shared memory (padded K-chunk stride).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe scripts/mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_nosw(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ inline uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void probe(int N, int ts, int nmma, int lbo, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 160 * 1024 / 4; i += blockDim.x) ((float*)smem)[i] = 0.001f * (i & 255);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(128, N);
    const uint32_t B0 = su32(smem), A0 = su32(smem + 80 * 1024);
    const uint64_t bd0 = desc_nosw(B0, lbo, 128), bstep = (uint64_t)((2 * lbo) >> 4);
    long long t0 = clock64();
    uint64_t bd = bd0;
    uint32_t acol = tmem;
    int s = 0;
#pragma unroll 17
    for (int i = 0; i < nmma; ++i) {
      const uint32_t acc = i ? 1u : 0u;
      if (ts) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem + 256),
            "r"(acol), "l"(bd), "r"(idesc), "r"(acc));
      } else {
        const uint64_t ad = desc_nosw(A0 + (uint32_t)(2 * s) * 2048, 2048, 128);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + 256),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      bd += bstep;
      acol += 8u;
      if (++s == 17) {
        s = 0;
        bd = bd0;
        acol = tmem;
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&mbar)));
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(su32(&mbar)), "r"(0));
    }
    long long t2 = clock64();
    out[blockIdx.x * 2 + 0] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

int main() {
  long long* d;
  cudaMalloc(&d, 2 * 148 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  long long h[2 * 148];
  for (int ts = 0; ts < 2; ++ts)
    for (int lbo : {528, 512, 1040})
      for (int N : {16, 32, 64, 128, 256}) {
        if (lbo == 1040 && N > 64) continue;
        const int nmma = 510;
        for (int rep = 0; rep < 2; ++rep) probe<<<1, 128, 160 * 1024>>>(N, ts, nmma, lbo, d);
        cudaMemcpy(h, d, 2 * sizeof(long long), cudaMemcpyDeviceToHost);
        cudaError_t e = cudaGetLastError();
        printf("%s N=%3d lbo=%4d: issue %.1f cyc/mma, complete %.1f cyc/mma  (%s)\n", ts ? "TS" : "SS", N, lbo,
               (double)h[0] / nmma, (double)h[1] / nmma, cudaGetErrorString(e));
      }
  // all SMs at once (TS, N = 32)
  for (int N : {32, 64, 128}) {
    probe<<<148, 128, 160 * 1024>>>(N, 1, 510, 528, d);
    cudaMemcpy(h, d, 2 * 148 * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[2 * i + 1] > mx ? h[2 * i + 1] : mx;
    printf("148 CTAs TS N=%d: max complete %.1f cyc/mma\n", N, (double)mx / 510);
  }
  return 0;
}
