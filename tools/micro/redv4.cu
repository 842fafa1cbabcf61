// Microbenchmark (SURVEY NEXT-1 evidence): throughput of the vectorised
// fire-and-forget reduction red.global.add.v4.f32 on B200 when the 32 lanes of
// a warp hit scattered 16-byte force slots (the j-side update of a half-list
// LJ sweep), against plain coalesced float4 stores for reference.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_red(float4 *f, const int *idx, int n, int iters) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int it = 0; it < iters; ++it) {
    const int j = idx[(i + it * 7919) % n];
    float *p = reinterpret_cast<float *>(f + j);
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(2.f),
                 "f"(3.f), "f"(4.f)
                 : "memory");
  }
}

__global__ void k_store(float4 *f, const int *idx, int n, int iters) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int it = 0; it < iters; ++it) {
    const int j = idx[(i + it * 7919) % n];
    f[j] = make_float4(1.f, 2.f, 3.f, (float)it);
  }
}

int main() {
  const int n = 1 << 20, iters = 36;
  int *h = new int[n];
  // neighbour-like locality: partner within +-2000 of i (cell-ordered particles)
  srand(1);
  for (int i = 0; i < n; ++i) {
    int j = i + (rand() % 4001) - 2000;
    h[i] = j < 0 ? j + n : (j >= n ? j - n : j);
  }
  int *idx;
  float4 *f;
  cudaMalloc(&idx, 4 * n);
  cudaMalloc(&f, 16 * n);
  cudaMemcpy(idx, h, 4 * n, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int k = 0; k < 2; ++k) {
    for (int mode = 0; mode < 2; ++mode) {
      cudaEventRecord(a);
      if (mode == 0) k_red<<<n / 256, 256>>>(f, idx, n, iters);
      else k_store<<<n / 256, 256>>>(f, idx, n, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)n * iters;
      printf("%s: %.3f ms for %.1fM scattered 16-byte ops = %.2f Gop/s\n",
             mode == 0 ? "red.global.add.v4.f32" : "st.global.v4 (plain)", ms, ops / 1e6,
             ops / (ms * 1e6));
    }
  }
  return 0;
}
