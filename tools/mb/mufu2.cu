// Microbenchmark (not product): MUFU ex2 throughput with independent accumulators (no FADD chain
// bound): f32, bf16 (per half), and f32 FFMA+MUFU+FADD mixes.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters) {
  float x[16], acc[16];
  for (int j = 0; j < 16; ++j) { x[j] = -(threadIdx.x * 0.001f + j * 0.1f); acc[j] = 0.f; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float e;
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x[j]));
      else {
        uint32_t r, a = __float_as_uint(x[j]) >> 16 | (__float_as_uint(x[j]) & 0xffff0000u);
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(a));
        e = __uint_as_float(r << 16);
      }
      acc[j] += e;
    }
  }
  float s = 0.f;
  for (int j = 0; j < 16; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 148, bs = 512, iters = 2048;
  float* o; cudaMalloc(&o, sms * 4 * bs * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int occ : {1, 2, 4}) {
    int g = sms * occ;
    double n = (double)g * bs * iters * 16;
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(a); k<0><<<g, bs>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (w) printf("occ %d CTAs x 512: ex2.f32        %8.2f MUFU lane-ops/clk/SM\n", occ, n / (ms * 1e-3) / sms / 1.965e9);
      cudaEventRecord(a); k<1><<<g, bs>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (w) printf("occ %d CTAs x 512: ex2.bf16x2 (per element, 2 MUFU/word) %8.2f elements/clk/SM\n", occ, 2 * n / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
