// Microbenchmark (not product): FAST-exit mass pass variants over a 64 KB bf16 row in smem.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
__device__ __forceinline__ uint32_t bfma2(uint32_t a, uint32_t b, uint32_t c) { uint32_t r; asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r; }
__device__ __forceinline__ uint32_t bex2(uint32_t a) { uint32_t r; asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(a)); return r; }
__device__ __forceinline__ float bacc2(float acc, uint32_t e) {
  asm("{\n .reg .b16 lo, hi;\n mov.b32 {lo, hi}, %1;\n add.rn.f32.bf16 %0, lo, %0;\n add.rn.f32.bf16 %0, hi, %0;\n}" : "+f"(acc) : "r"(e)); return acc; }
__device__ __forceinline__ float ex2f(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int MODE>
__global__ void __launch_bounds__(480, 1) k(int reps, float* out) {
  extern __shared__ uint4 R[];
  for (int i = threadIdx.x; i < 4000; i += 480) R[i] = make_uint4(0xc0a0bf80u + i, 0x40003f00u ^ i, 0xbf00c100u + i, 0x3e80c0c0u);
  __syncthreads();
  const uint32_t L2 = 0x40194019u;
  float tot = 0.f;
  for (int r = 0; r < reps; ++r) {
    const uint32_t nm = 0xc1c8c1c8u ^ (r & 7) ^ ((r & 7) << 16);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    for (int v = threadIdx.x; v < 4000; v += 480) {
      uint4 q = R[v];
      if (MODE == 0) {  // current: one accumulator
        a0 = bacc2(a0, bex2(bfma2(q.x, L2, nm))); a0 = bacc2(a0, bex2(bfma2(q.y, L2, nm)));
        a0 = bacc2(a0, bex2(bfma2(q.z, L2, nm))); a0 = bacc2(a0, bex2(bfma2(q.w, L2, nm)));
      } else if (MODE == 1) {  // four accumulators
        a0 = bacc2(a0, bex2(bfma2(q.x, L2, nm))); a1 = bacc2(a1, bex2(bfma2(q.y, L2, nm)));
        a2 = bacc2(a2, bex2(bfma2(q.z, L2, nm))); a3 = bacc2(a3, bex2(bfma2(q.w, L2, nm)));
      } else if (MODE == 2) {  // bf16x2 exps, packed bf16x2 add tree of 4 then fp32
        uint32_t e0 = bex2(bfma2(q.x, L2, nm)), e1 = bex2(bfma2(q.y, L2, nm)), e2 = bex2(bfma2(q.z, L2, nm)), e3 = bex2(bfma2(q.w, L2, nm));
        float s0 = __uint_as_float(e0 << 16) + __uint_as_float(e0 & 0xffff0000u);
        float s1 = __uint_as_float(e1 << 16) + __uint_as_float(e1 & 0xffff0000u);
        float s2 = __uint_as_float(e2 << 16) + __uint_as_float(e2 & 0xffff0000u);
        float s3 = __uint_as_float(e3 << 16) + __uint_as_float(e3 & 0xffff0000u);
        a0 += (s0 + s1) + (s2 + s3);
      } else if (MODE == 3) {  // fp32: unpack, FFMA, MUFU f32, FADD
        uint32_t w[4] = {q.x, q.y, q.z, q.w};
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) { float z = (j & 1) ? __uint_as_float(w[j >> 1] & 0xffff0000u) : __uint_as_float(w[j >> 1] << 16); s += ex2f(fmaf(z, 2.4f, -25.f - (float)(r & 7))); }
        a0 += s;
      } else if (MODE == 4) {  // loads only
        a0 += __uint_as_float(q.x ^ nm) + __uint_as_float(q.w);
      }
    }
    tot += a0 + a1 + a2 + a3;
  }
  if (tot == 1.2345f) out[0] = tot;
}
int main() {
  float* o; cudaMalloc(&o, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int reps = 2000;
  auto run = [&](auto kern, const char* n) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64000);
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(a); kern<<<148, 480, 64000>>>(reps, o); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (w) printf("%-40s %.3f ms  %.0f clks per 32000-elem row per SM  %s\n", n, ms, ms * 1e-3 * 1.965e9 / reps, cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(k<0>, "bf16 ex2, one acc (current)");
  run(k<1>, "bf16 ex2, four accs");
  run(k<2>, "bf16 ex2, fp32 tree");
  run(k<3>, "fp32 FFMA + MUFU f32");
  run(k<4>, "loads only");
}
