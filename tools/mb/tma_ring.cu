// Microbenchmark (not product): HBM streaming through a TMA bulk-copy smem ring.
// One persistent CTA per SM, producer lane + consumer warps; rows of ROWB bytes
// loaded as NSPLIT bulk copies into STAGES buffers; consumers optionally read the
// row from smem (pass A-like max) before releasing the stage.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(unsigned long long* b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(su(b)), "r"(ph) : "memory");
}
template <int STAGES, int NSPLIT, int READ>
__global__ void __launch_bounds__(512, 1) ring(const char* rows, int nrows, int rowb, int* next, float* out) {
  extern __shared__ __align__(128) unsigned char raw[];
  unsigned long long* full = (unsigned long long*)raw;
  unsigned long long* empty = full + STAGES;
  int* stask = (int*)(empty + STAGES);
  char* buf = (char*)raw + 1024;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 15) {
    if (lane == 0) {
      for (int it = 0;; ++it) {
        int s = it % STAGES, k = it / STAGES;
        if (k > 0) wait(&empty[s], (k - 1) & 1);
        int t = atomicAdd(next, 1);
        if (t >= nrows) { stask[s] = -1; asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&full[s])) : "memory"); break; }
        stask[s] = t;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(rowb) : "memory");
        for (int p = 0; p < NSPLIT; ++p) {
          int cb = rowb / NSPLIT;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(buf + (size_t)s * rowb + p * cb)),
                       "l"(rows + (size_t)t * rowb + p * cb), "r"(cb), "r"(su(&full[s])) : "memory");
        }
      }
    }
    return;
  }
  float acc = 0.f;
  for (int it = 0;; ++it) {
    int s = it % STAGES;
    wait(&full[s], (it / STAGES) & 1);
    if (stask[s] < 0) break;
    if (READ) {
      const uint4* R = (const uint4*)(buf + (size_t)s * rowb);
      for (int v = tid; v < rowb / 16; v += 480) { uint4 q = R[v]; acc += __uint_as_float(q.x) + __uint_as_float(q.w); }
    }
    asm volatile("bar.sync 1, 480;" ::: "memory");
    if (tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
  }
  if (acc == 12345.f) out[0] = acc;
}

template <int STAGES, int NSPLIT, int READ>
void run(const char* rows, int nrows, int rowb, int* next, float* out, const char* name) {
  size_t smem = 1024 + (size_t)STAGES * rowb;
  cudaFuncSetAttribute(ring<STAGES, NSPLIT, READ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaMemset(next, 0, 4);
    cudaEventRecord(a);
    ring<STAGES, NSPLIT, READ><<<148, 512, smem>>>(rows, nrows, rowb, next, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  printf("%-34s rowB=%6d  %8.3f ms  %7.1f GB/s  %s\n", name, rowb, best, (double)nrows * rowb / best / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  size_t total = (size_t)4 << 30;
  char* rows; cudaMalloc(&rows, total); cudaMemset(rows, 1, total);
  int* next; cudaMalloc(&next, 4); float* out; cudaMalloc(&out, 4);
  int rb = 64000, n = (int)(total / rb);
  run<3, 1, 0>(rows, n, rb, next, out, "3 stages x 1 copy, no read");
  run<3, 4, 0>(rows, n, rb, next, out, "3 stages x 4 copies, no read");
  run<3, 1, 1>(rows, n, rb, next, out, "3 stages x 1 copy, read");
  run<3, 4, 1>(rows, n, rb, next, out, "3 stages x 4 copies, read");
  int rb2 = 32000; int n2 = (int)(total / rb2);
  run<6, 1, 0>(rows, n2, rb2, next, out, "6 stages x 32KB, no read");
  run<6, 1, 1>(rows, n2, rb2, next, out, "6 stages x 32KB, read");
  int rb3 = 16000; int n3 = (int)(total / rb3);
  run<12, 1, 0>(rows, n3, rb3, next, out, "12 stages x 16KB, no read");
  // plain copy reference
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); cudaMemcpy(rows + total / 2, rows, total / 2, cudaMemcpyDeviceToDevice); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); printf("memcpy d2d r+w %.1f GB/s\n", (double)total / ms / 1e6);
}
