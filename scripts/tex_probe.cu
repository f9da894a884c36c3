// Throughput probe: trilinear ring samples through two tld4 (tex2Dgather) texture gathers per sample vs eight
// shared-memory loads per sample (the stage-1 sampler's inner loop, isolated).  Prints samples/s for both.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tex_probe scripts/tex_probe.cu
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

constexpr int N = 64, NP = 15, W = N + 8;
constexpr int kRings = 2048;  // rings per CTA

__device__ __forceinline__ float lerp(float a, float b, float f) { return fmaf(f, b - a, a); }

__global__ void __launch_bounds__(512) k_tex(cudaTextureObject_t t, float* out) {
  float acc = 0.f;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = warp; r < kRings; r += 16) {
    const int p = (blockIdx.x + r) % NP;
    const int z0 = 8 + (r * 7) % 48;
    const float rad = 4.0f + (r % 28), fz = 0.37f;
    const float rowbase = (float)(p * N * N + z0 * N) + 1.0f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float s, c;
      __sincosf(0.0245f * (lane + 32 * q) + 0.001f * r, &s, &c);
      const float px = 31.5f + rad * c, py = 31.5f + rad * s;
      const float fx0 = floorf(px), fy0 = floorf(py);
      const float fx = px - fx0, fy = py - fy0;
      const float4 a = tex2Dgather<float4>(t, fx0 + 1.0f, rowbase + fy0, 0);
      const float4 b = tex2Dgather<float4>(t, fx0 + 1.0f, rowbase + fy0 + N, 0);
      // order: x = (x0, y0+1), y = (x0+1, y0+1), z = (x0+1, y0), w = (x0, y0)
      const float c0 = lerp(lerp(a.w, a.z, fx), lerp(a.x, a.y, fx), fy);
      const float c1 = lerp(lerp(b.w, b.z, fx), lerp(b.x, b.y, fx), fy);
      acc += lerp(c0, c1, fz);
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void __launch_bounds__(512) k_smem(const float* vol, float* out) {
  extern __shared__ float pl[];  // 2 planes [N][W]
  for (int t = threadIdx.x; t < 2 * N * W; t += blockDim.x) pl[t] = vol[t % (N * N)];
  __syncthreads();
  float acc = 0.f;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = warp; r < kRings; r += 16) {
    const float rad = 4.0f + (r % 28), fz = 0.37f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float s, c;
      __sincosf(0.0245f * (lane + 32 * q) + 0.001f * r, &s, &c);
      const float px = 31.5f + rad * c, py = 31.5f + rad * s;
      const float fx0 = floorf(px), fy0 = floorf(py);
      const float fx = px - fx0, fy = py - fy0;
      const float* b = pl + (int)fy0 * W + (int)fx0;
      const float c0 = lerp(lerp(b[0], b[1], fx), lerp(b[W], b[W + 1], fx), fy);
      const float* b1 = b + N * W;
      const float c1 = lerp(lerp(b1[0], b1[1], fx), lerp(b1[W], b1[W + 1], fx), fy);
      acc += lerp(c0, c1, fz);
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const size_t n = (size_t)NP * N * N * N;
  float* d;
  cudaMalloc(&d, n * 4);
  cudaMemset(d, 0, n * 4);
  cudaResourceDesc rd;
  memset(&rd, 0, sizeof(rd));
  rd.resType = cudaResourceTypePitch2D;
  rd.res.pitch2D.devPtr = d;
  rd.res.pitch2D.desc = cudaCreateChannelDesc<float>();
  rd.res.pitch2D.width = N;
  rd.res.pitch2D.height = (size_t)NP * N * N;
  rd.res.pitch2D.pitchInBytes = N * 4;
  cudaTextureDesc td;
  memset(&td, 0, sizeof(td));
  td.addressMode[0] = td.addressMode[1] = cudaAddressModeBorder;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t t;
  printf("create %d\n", (int)cudaCreateTextureObject(&t, &rd, &td, nullptr));
  float* o;
  cudaMalloc(&o, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t smem = 2 * N * W * 4;
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int blocksPerSm = 1; blocksPerSm <= 2; ++blocksPerSm) {
    const int grid = sms * blocksPerSm * 8;
    const double samples = (double)grid * kRings * 32 * 4;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_tex<<<grid, 512>>>(t, o);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("tex  grid %d: %.3f ms  %.1f G samples/s\n", grid, ms, samples / ms / 1e6);
      cudaEventRecord(e0);
      k_smem<<<grid, 512, smem>>>(d, o);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("smem grid %d: %.3f ms  %.1f G samples/s\n", grid, ms, samples / ms / 1e6);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
