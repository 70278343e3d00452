// Task plumbing and FAST exponentials shared by the resample kernels
// (lc_resample.cu: row-warp / CTA / EXACT tiers; lc_stage.cu: smem-staged rows).
#pragma once
#include <float.h>
#include <limits.h>
#include <math.h>

#include "lc_common.cuh"

namespace lcb {

// ---- error model ----------------------------------------------
// ex2.approx.ftz.f32 relative error bound (PTX ISA: ~2 ulp).  The GPU test
// tests/test_gpu_parity.py::test_fast_exp_error_bound measures fast_exp over
// dense argument grids and fails if this constant is ever exceeded.
constexpr double kEx2RelErr = 4.0e-7;    // fast_exp (corrected) incl. margin
constexpr double kEx2Raw = 2.5e-7;       // ex2.approx.ftz.f32 alone (cheap_exp), measured bound + margin
constexpr double kArgRel = 3.0 * 5.9604644775390625e-08 * 0.6931471805599453 * 1.01;  // cheap_exp: per |a|
constexpr double kCorrErr = 1.0e-10;                       // 2nd-order term of the argument correction
constexpr double kSum8Err = 3.0 * 5.9604644775390625e-08;  // fp32 pairwise sum of 8 (3 roundings)
constexpr double kSum16Err = 4.0 * 5.9604644775390625e-08;  // fp32 pairwise sum of 16 (4 roundings)
constexpr double kRefExpErr = 8.881784197001252e-16;       // libm / numpy exp vs exact: 4 ulp
constexpr double kLiteErr = 3.0e-13;                       // lite_exp incl. its argument (|a| <= 1100)
constexpr double kEps64 = 1.1102230246251565e-16;          // 2^-53

// ---- exponentials ------------------------------------------------------------------------------

struct ExpCtx {
  float m;         // row max (exact)
  float Lhi, Llo;  // log2(e)/T split, Lhi + Llo = log2e/T to ~2^-48
  double T;
  double mT;       // fl(m / T): the reference's scaled max (sampling.py:65-66)
  double md;       // (double) m
  double L16;      // 16 * log2(e) / T
};

// FAST: e ~ 2^((z-m) * log2e / T).  z - m is carried exactly (TwoSum), the
// product error and the constant's low part go into alo, and ex2's input
// rounding is removed by the first-order correction e*(1 + alo*ln2).
// Relative error <= kEx2RelErr + kCorrErr; 0 for z = -inf; e(m) == 1 exactly.
__device__ __forceinline__ float fast_exp(const ExpCtx& c, float z) {
  float s = z - c.m;
  float bb = s - z;
  float err = (z - (s - bb)) + (-c.m - bb);
  float ahi = s * c.Lhi;
  float alo = fmaf(s, c.Lhi, -ahi) + fmaf(err, c.Lhi, s * c.Llo);
  float e = ex2_approx(ahi);
  return (e > 0.0f) ? fmaf(e, alo * 0.69314718055994531f, e) : 0.0f;
}

// fast_exp of two elements with packed pair instructions: the same IEEE operations in the same
// order per lane (bit-identical to two fast_exp calls), about half the FP32 instructions
__device__ __forceinline__ float2 fast_exp2(float m, float Lhi, float Llo, float2 z) {
  const float2 M = make_float2(m, m), nM = make_float2(-m, -m);
  const float2 H = make_float2(Lhi, Lhi), Lo = make_float2(Llo, Llo);
  const float2 s = f2sub(z, M);
  const float2 bb = f2sub(s, z);
  const float2 err = f2add(f2sub(z, f2sub(s, bb)), f2sub(nM, bb));
  const float2 ahi = f2mul(s, H);
  const float2 nahi = make_float2(-ahi.x, -ahi.y);
  const float2 alo = f2add(f2fma(s, H, nahi), f2fma(err, H, f2mul(s, Lo)));
  const float2 e = make_float2(ex2_approx(ahi.x), ex2_approx(ahi.y));
  const float2 r = f2fma(e, f2mul(alo, make_float2(0.69314718055994531f, 0.69314718055994531f)), e);
  return make_float2(e.x > 0.0f ? r.x : 0.0f, e.y > 0.0f ? r.y : 0.0f);
}

// CHEAP (truncated modes, where only the row mass and bracketing use it):
// e = ex2(fl(fl(z - m) * Lhi)).  Relative error <= kEx2Raw + kArgRel * |a|
// (three fp32 roundings carried into the argument); a is clamped at -200 so
// -inf inputs give e = 0 and e*a = 0.
__device__ __forceinline__ float cheap_exp(const ExpCtx& c, float z, float& a) {
  a = fmaxf((z - c.m) * c.Lhi, -200.0f);
  return ex2_approx(a);
}

// PRECISE: table-driven fp64 exp of (z - m)/T.  b = 16*log2e*(z-m)/T,
// n = rint(b), x = b - n in [-1/2, 1/2]; 2^(b/16) = 2^(n>>4) * 2^((n&15)/16) *
// exp(x*ln2/16) with a degree-6 Taylor polynomial (|x ln2/16| <= 0.0217,
// truncation 5e-16).  Relative error <= kLiteErr for |b/16| <= 1100.
__device__ __forceinline__ double lite_exp(const ExpCtx& c, float z, const double* t16) {
  const double b = ((double)z - c.md) * c.L16;
  if (!(b > -17000.0)) return 0.0;
  const double t = b + 6755399441055744.0;  // 1.5 * 2^52: round to nearest
  const int n16 = __double2loint(t);
  const double x = b - (t - 6755399441055744.0);
  double p = 9.181219573844438764e-12;
  p = fma(x, p, 1.271587195055813162e-9);
  p = fma(x, p, 1.467610032291942926e-7);
  p = fma(x, p, 1.355080777949745604e-5);
  p = fma(x, p, 9.383847928089871576e-4);
  p = fma(x, p, 4.332169878499658184e-2);
  p = fma(x, p, 1.0);
  const double r = t16[n16 & 15] * p;
  const int e2 = n16 >> 4;
  if (e2 >= -1021) return __hiloint2double(__double2hiint(r) + (e2 << 20), __double2loint(r));
  return (r * __hiloint2double((e2 + 1023 + 600) << 20, 0)) * 0x1p-600;
}

__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
// 3-input forms (sm_100 FMNMX3): max.NaN propagates NaN like max_nan, min like fminf
__device__ __forceinline__ float max3_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float min3f(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float min_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// ---- task plumbing ------------------------------------------------------------------------------

struct TaskView {
  const char* row;
  int V;
  double T;
  double Ld;  // log2(e) / T (0 when T == 0), computed once per task by whoever resolves it
  int topk;  // effective top-k (0 = none / k >= V)
  double topp;
  bool trunc;
  int64_t d0, d1;
  int64_t seed_base;
  int64_t u_index;
};

struct CacheMap {
  const int32_t* pages;  // [slots][max_pages], -1 = unused
  int max_pages;
  int page_rows;
};

struct DrawIO {
  const double* u;
  const uint64_t* seed;
  const int64_t* index;
  int32_t* token;
  uint8_t* flags;
  int32_t* kept;  // per task |kept| (lc_draws.d_kept), may be null
};

// the kept-set size of task t (first K ids in (z desc, id asc) order), when requested
__device__ __forceinline__ void set_kept(const DrawIO& io, int t, int K) {
  if (io.kept) io.kept[t] = K;
}
// |kept_order| of the one-hot softmax at T == 0 (sampling.py:61-64 then :71-94): the argmax
// alone under a nucleus, else the top-k prefix (argmax + zero-probability ids), else identity
__device__ __forceinline__ int greedy_kept(int V, int topk, double topp) {
  return topp < 1.0 ? 1 : (topk > 0 ? topk : V);
}

struct Workspace {
  int* q_exact;   // [0] = count, [1..] task ids
  int* q_cta;     // tasks the row-warp kernel hands to the CTA kernel (same layout)
  int* scr_id;    // [grid][2][SCR_PER_CTA]
  double* scr_e;  // [grid][2][SCR_PER_CTA]
};

__device__ __forceinline__ double draw_u(const DrawIO& io, int64_t d, const TaskView& tv) {
  if (io.u) return io.u[d];
  if (io.index) return request_uniform(io.seed[d], (uint64_t)io.index[d]);
  return request_uniform(io.seed[tv.seed_base + (d - tv.d0)], (uint64_t)tv.u_index);
}

__device__ __forceinline__ bool resolve_task(const lc_task& tk, const char* rows, int64_t row_bytes, int Vdef,
                                             const CacheMap& cm, TaskView& tv) {
  tv.d0 = tk.draw_begin;
  tv.d1 = tk.draw_end;
  tv.seed_base = tk.seed_base;
  tv.u_index = tk.u_index >= 0 ? tk.u_index : tk.pos;
  tv.V = tk.vocab > 0 ? tk.vocab : Vdef;
  tv.T = tk.temperature;
  tv.Ld = tv.T > 0.0 ? 1.4426950408889634 / tv.T : 0.0;
  tv.topk = (tk.top_k > 0 && tk.top_k < tv.V) ? tk.top_k : 0;
  tv.topp = tk.top_p;
  tv.trunc = !(tk.top_k <= 0 && tk.top_p == 1.0);
  tv.row = nullptr;
  if (tv.V < 1 || tv.V > Vdef || !(tv.T >= 0.0) || !(tv.topp > 0.0 && tv.topp <= 1.0)) return false;
  int64_t r = tk.row;
  if (r < 0) {
    if (!cm.pages || tk.slot < 0 || tk.pos < 0) return false;
    int pg = tk.pos / cm.page_rows;
    if (pg >= cm.max_pages) return false;
    int page = cm.pages[(int64_t)tk.slot * cm.max_pages + pg];
    if (page < 0) return false;
    r = (int64_t)page * cm.page_rows + tk.pos % cm.page_rows;
  }
  tv.row = rows + r * row_bytes;
  return true;
}

__device__ __forceinline__ void write_all(const TaskView& tv, const DrawIO& io, int tok, uint8_t flag) {
  for (int64_t d = tv.d0 + threadIdx.x; d < tv.d1; d += blockDim.x) {
    io.token[d] = tok;
    if (io.flags) io.flags[d] = flag;
  }
}

// smem-staged kernel (lc_stage.cu): bf16 rows of <= 32768 ids, TMA-loaded
bool stage_eligible(int dtype, int64_t V, int64_t row_bytes, const void* rows);
int stage_launch(const char* rows, int64_t row_bytes, int V, const lc_task* tasks, int64_t n_tasks, CacheMap cm,
                 DrawIO io, int* next, int* q_cta, unsigned long long* counters, int n_sms, cudaStream_t st);

unsigned long long* stage_prof_buffer();
// wide top-k kernel (lc_wide.cu): bf16 rows wider than 32000 ids with top-k <= 64
bool wide_eligible(int dtype, int64_t V, int64_t row_bytes, const void* rows);
int wide_launch(const char* rows, int64_t row_bytes, int V, const lc_task* tasks, int64_t n_tasks, CacheMap cm,
                DrawIO io, int* next, int* q_cta, unsigned long long* counters, int n_sms, cudaStream_t st);

}  // namespace lcb
