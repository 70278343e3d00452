// Shared pieces of the TMA-staged resample kernels (lc_stage.cu: bf16 rows with a
// nucleus; lc_wide.cu: top-k rows of any width): PTX wrappers (mbarrier, bulk copy,
// packed bf16), task plumbing and the producer -> group task FIFO.
#pragma once
#include "lc_common.cuh"
#include "lc_task.cuh"

namespace lcb {

// ---- PTX helpers ------------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// bulk prefetch of [src, src + bytes) into L2 (no completion tracking)
__device__ __forceinline__ void l2_prefetch(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// named barrier of group g (ids 1..groups), NT threads
template <int NT>
__device__ __forceinline__ void gbar_n(int g) { asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "n"(NT) : "memory"); }

__device__ __forceinline__ uint32_t bmax2_nan(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t bfma2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t bex2(uint32_t a) {
  uint32_t r;
  asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(a));
  return r;
}
// acc + lo(e) + hi(e), the bf16 halves added straight into fp32 (FHADD.BF16)
__device__ __forceinline__ float bacc2(float acc, uint32_t e) {
  asm("{\n .reg .b16 lo, hi;\n mov.b32 {lo, hi}, %1;\n add.rn.f32.bf16 %0, lo, %0;\n add.rn.f32.bf16 %0, hi, %0;\n}"
      : "+f"(acc)
      : "r"(e));
  return acc;
}
__device__ __forceinline__ uint32_t badd2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// acc + ex2(lo(a)) + ex2(hi(a)): the two bf16 exponentials (MUFU.EX2.BF16 per half) added straight
// into fp32 (FHADD.BF16) -- no repacking of the halves, no bf16 rounding of pair sums
__device__ __forceinline__ float bex2_acc(float acc, uint32_t a) {
  asm("{\n .reg .b16 l, h, el, eh;\n mov.b32 {l, h}, %1;\n ex2.approx.ftz.bf16 el, l;\n ex2.approx.ftz.bf16 eh, h;\n"
      " add.rn.f32.bf16 %0, el, %0;\n add.rn.f32.bf16 %0, eh, %0;\n}"
      : "+f"(acc)
      : "r"(a));
  return acc;
}
// acc + lo(e) / acc + hi(e): one bf16 half added straight into fp32 (FHADD.BF16)
__device__ __forceinline__ float bacc_lo(float acc, uint32_t e) {
  asm("{\n .reg .b16 lo, hi;\n mov.b32 {lo, hi}, %1;\n add.rn.f32.bf16 %0, lo, %0;\n}" : "+f"(acc) : "r"(e));
  return acc;
}
__device__ __forceinline__ float bacc_hi(float acc, uint32_t e) {
  asm("{\n .reg .b16 lo, hi;\n mov.b32 {lo, hi}, %1;\n add.rn.f32.bf16 %0, hi, %0;\n}" : "+f"(acc) : "r"(e));
  return acc;
}
__device__ __forceinline__ uint32_t bf16_bits(float f) { return (uint32_t)f32_to_bf16_bits(f); }
__device__ __forceinline__ float lo_f(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi_f(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
// order key of a bf16 value given as fp32 bits (larger value -> larger key; -0 < +0)
__device__ __forceinline__ uint32_t key16(uint32_t fbits) {
  return (fbits ^ ((uint32_t)((int32_t)fbits >> 31) | 0x80000000u)) >> 16;
}
__device__ __forceinline__ float key16_to_f(uint32_t k) {
  const uint32_t h = (k & 0x8000u) ? (k & 0x7fffu) : (~k & 0xffffu);
  return __uint_as_float(h << 16);
}
// the low half zero-extended by a byte permute (PRMT): kept apart from the shift that follows, so
// base + (lo << s) is one LEA instead of shift + mask + add
__device__ __forceinline__ uint32_t lo16(uint32_t w) { return __byte_perm(w, 0u, 0x4410); }
__device__ __forceinline__ uint32_t off_lo(uint32_t w) { return w & 0xffffu; }
__device__ __forceinline__ uint32_t off_hi(uint32_t w) { return w >> 16; }

// predicated shared-memory increment / fp64 gather-add, branch-free (no BSSY/BSYNC
// around each element)
__device__ __forceinline__ void pinc(uint32_t* addr, bool p) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n @q red.shared.add.u32 [%0], 1;\n}" ::"r"(smem_u32(addr)),
      "r"((uint32_t)p)
      : "memory");
}
__device__ __forceinline__ double pgather(const double* base, uint32_t idx, bool p) {
  double r;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n mov.f64 %0, 0d0000000000000000;\n @q ld.shared.f64 %0, [%1];\n}"
      : "=d"(r)
      : "r"(smem_u32(base) + 8u * idx), "r"((uint32_t)p));
  return r;
}

// the same gather without `volatile`: the compiler may batch independent gathers ahead of their
// uses (the table must not change between the caller's last barrier and the gather)
__device__ __forceinline__ double pgather_nv(const double* base, uint32_t idx, bool p) {
  double r;
  asm("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n mov.f64 %0, 0d0000000000000000;\n @q ld.shared.f64 %0, [%1];\n}"
      : "=d"(r)
      : "r"(smem_u32(base) + 8u * idx), "r"((uint32_t)p));
  return r;
}

// ---- the kernel --------------------------------------------------------------------------------

struct StageArgs {
  const char* rows;
  int64_t row_bytes;
  int Vdef;
  const lc_task* tasks;
  int n_tasks;
  CacheMap cm;
  DrawIO io;
  int* next;   // dynamic task counter
  int* q_cta;  // requeue: [0] count, [1..] task ids (CTA kernel)
  unsigned long long* counters;
  unsigned long long* prof;  // optional per-phase clock totals (LCB_STAGE_PROF=1)
};

__device__ __forceinline__ void requeue(const StageArgs& a, int task_id) {
  const int pos = atomicAdd(a.q_cta, 1);
  a.q_cta[1 + pos] = task_id;
}

__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

// CTA-scope acquire load / release store of a shared int (the task FIFO's indices): lighter than a
// sequentially consistent __threadfence_block() around volatile accesses
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// one 4-byte word per lane (lanes 0 .. sizeof(T)/4 - 1)
template <typename T>
__device__ __forceinline__ void warp_copy(T& dst, const T& src, int lane) {
  static_assert(sizeof(T) % 4 == 0 && sizeof(T) <= 128, "warp_copy");
  if (lane < (int)(sizeof(T) / 4))
    reinterpret_cast<uint32_t*>(&dst)[lane] = reinterpret_cast<const uint32_t*>(&src)[lane];
}


}  // namespace lcb
