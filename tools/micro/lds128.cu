// Microbenchmark: cycles per LDS.128 (warp) for several lane->slot patterns,
// to check the quarter-warp bank-group conflict model on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const int *pat, int iters, float4 *out, long long *cyc) {
  __shared__ float4 s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, 1, 2, 3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int idx[8];
  for (int u = 0; u < 8; ++u) idx[u] = pat[u * 32 + lane];
  float4 acc = make_float4(0, 0, 0, 0);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float4 v = s[idx[u]];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      idx[u] += (int)v.w - 3;
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  int h[8 * 32];
  const char *names[] = {"contiguous", "same-group stride8", "random", "quarter-distinct-groups", "broadcast"};
  srand(1);
  for (int p = 0; p < 5; ++p) {
    for (int u = 0; u < 8; ++u)
      for (int l = 0; l < 32; ++l) {
        int v;
        if (p == 0) v = u * 32 + l;
        else if (p == 1) v = (u * 32 + l) * 8 % 2048;
        else if (p == 2) v = rand() % 2048;
        else if (p == 3) v = ((rand() % 250) * 8 + ((l & 7) + u) % 8);  // distinct groups per quarter
        else v = u;
        h[u * 32 + l] = v;
      }
    int *d; float4 *o; long long *c, hc;
    cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 148 * 8 * 256 * 16); cudaMalloc(&c, 8);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int warps = 1; warps <= 32; warps *= 4) {
      int iters = 2000;
      k<<<1, warps * 32>>>(d, iters, o, c);
      cudaDeviceSynchronize();
      cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
      printf("%-26s warps/SM %2d: %.2f cycles per LDS.128 (SM-wide)\n", names[p], warps,
             (double)hc / (iters * 8.0 * warps));
    }
    cudaFree(d); cudaFree(o); cudaFree(c);
  }
  return 0;
}
