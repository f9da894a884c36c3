// Probe of the tex2Dgather (tld4) component order on this GPU: texel (x, y) holds 10 y + x.
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
__global__ void k(cudaTextureObject_t t, float4* o) {
  o[0] = tex2Dgather<float4>(t, 2.0f, 2.0f, 0);   // footprint x0 = 1, y0 = 1
  o[1] = tex2Dgather<float4>(t, 0.0f, 1.0f, 0);   // x0 = -1 (border), y0 = 0
}
int main() {
  const int W = 8, Hh = 8;
  float h[W * Hh];
  for (int y = 0; y < Hh; ++y) for (int x = 0; x < W; ++x) h[y * W + x] = 10 * y + x + 1;
  float* d; cudaMalloc(&d, sizeof(h)); cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaResourceDesc rd; memset(&rd, 0, sizeof(rd));
  rd.resType = cudaResourceTypePitch2D; rd.res.pitch2D.devPtr = d; rd.res.pitch2D.desc = cudaCreateChannelDesc<float>();
  rd.res.pitch2D.width = W; rd.res.pitch2D.height = Hh; rd.res.pitch2D.pitchInBytes = W * 4;
  cudaTextureDesc td; memset(&td, 0, sizeof(td));
  td.addressMode[0] = td.addressMode[1] = cudaAddressModeBorder; td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t t; printf("create %d\n", (int)cudaCreateTextureObject(&t, &rd, &td, nullptr));
  float4* o; cudaMalloc(&o, 2 * sizeof(float4)); k<<<1, 1>>>(t, o); float4 r[2];
  cudaMemcpy(r, o, sizeof(r), cudaMemcpyDeviceToHost);
  printf("gather(x0=1,y0=1): %g %g %g %g   [(x,y) -> 10y+x+1]\n", r[0].x, r[0].y, r[0].z, r[0].w);
  printf("gather(x0=-1,y0=0): %g %g %g %g\n", r[1].x, r[1].y, r[1].z, r[1].w);
  return 0;
}
