// Microbenchmarks (not product): MUFU ex2 variants, smem atomics / gathers.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__global__ void ex2_f32(float* out, int iters) {
  float x[8];
  for (int j = 0; j < 8; ++j) x[j] = -(threadIdx.x * 0.001f + j * 0.1f);
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { float e; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x[j])); acc += e; x[j] -= 1e-7f; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void ex2_f16(float* out, int iters) {
  uint32_t x[8];
  for (int j = 0; j < 8; ++j) x[j] = 0xbc00bc00u + j + threadIdx.x;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { uint32_t e; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(e) : "r"(x[j])); acc ^= e; x[j] += 1; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}
__global__ void ex2_bf16(float* out, int iters) {
  uint32_t x[8];
  for (int j = 0; j < 8; ++j) x[j] = 0xbf80bf80u + j + threadIdx.x;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { uint32_t e; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(e) : "r"(x[j])); acc ^= e; x[j] += 1; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}
__global__ void atoms_hist(float* out, int iters, int nbins) {
  __shared__ uint32_t h[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t s = threadIdx.x * 2654435761u + blockIdx.x;
  for (int i = 0; i < iters; ++i) { s = s * 1664525u + 1013904223u;
#pragma unroll
    for (int j = 0; j < 8; ++j) { atomicAdd(&h[(s + j * 2654435761u) >> 20 & (nbins - 1)], 1u); }
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = h[threadIdx.x];
}
__global__ void lds_gather(float* out, int iters, int nbins) {
  __shared__ double t[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) t[i] = i;
  __syncthreads();
  uint32_t s = threadIdx.x * 2654435761u + blockIdx.x;
  double acc = 0;
  for (int i = 0; i < iters; ++i) { s = s * 1664525u + 1013904223u;
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc += t[(s + j * 2654435761u) >> 20 & (nbins - 1)]; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void alu_only(float* out, int iters, int nbins) {
  uint32_t s = threadIdx.x * 2654435761u + blockIdx.x; uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) { s = s * 1664525u + 1013904223u;
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc += (s + j * 2654435761u) >> 20 & (nbins - 1); }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms = 148, bs = 512, iters = 4096;
  float* o; cudaMalloc(&o, sms * 4 * bs * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  auto rep = [&](const char* n, double ops) {
    cudaEventElapsedTime(&ms, a, b);
    printf("%-28s %8.3f ms  %8.2f ops/clk/SM (at 1.965GHz)\n", n, ms, ops / (ms * 1e-3) / sms / 1.965e9);
  };
  int g = sms * 2;
  double n = (double)g * bs * iters * 8;
  for (int w = 0; w < 2; ++w) {
    cudaEventRecord(a); ex2_f32<<<g, bs>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b); if (w) rep("ex2.f32", n);
    cudaEventRecord(a); ex2_f16<<<g, bs>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b); if (w) rep("ex2.f16x2 (elements)", 2 * n);
    cudaEventRecord(a); ex2_bf16<<<g, bs>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b); if (w) rep("ex2.bf16x2 (elements)", 2 * n);
    for (int nb : {64, 512, 2048, 4096}) {
      char buf[64];
      cudaEventRecord(a); atoms_hist<<<g, bs>>>(o, iters / 4, nb); cudaEventRecord(b); cudaEventSynchronize(b);
      snprintf(buf, 64, "atoms nbins=%d", nb); if (w) rep(buf, n / 4);
      cudaEventRecord(a); lds_gather<<<g, bs>>>(o, iters / 4, nb); cudaEventRecord(b); cudaEventSynchronize(b);
      snprintf(buf, 64, "lds64 gather nbins=%d", nb); if (w) rep(buf, n / 4);
    }
    cudaEventRecord(a); alu_only<<<g, bs>>>(o, iters / 4, 2048); cudaEventRecord(b); cudaEventSynchronize(b); if (w) rep("alu only (lcg)", n / 4);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
