// K1: fused temperature -> softmax -> top-k/top-p -> inverse-CDF draw.
//
// Reference semantics (bit-exact token decisions given the same uniform):
//   softmax   sampling.py:57-68   s = f64(z)/T - max, e = exp(s), p = e / pairwise_sum(e)
//   truncate  sampling.py:71-94   order (p desc, id asc); top-k if k < V; nucleus on the
//                                 UNtruncated mass: cut = first csum >= top_p ('left');
//                                 renormalise by the kept sum
//   sample    sampling.py:97-109  t = u * pairwise_sum(q); first id with cumsum(q) > t
//                                 ('right'), clamp to V-1, back off over q == 0
//
// Tiers:
//   FAST     fp32 MUFU exponentials with an exactly-carried argument and a
//            rigorous per-row error bound; every decision (nucleus cut, draw) is
//            certified against the bound.
//   PRECISE  (same CTA, same task, second pass) only when a FAST decision is
//            uncertain: the row mass is recomputed with a table-driven fp64
//            exponential (~12 fp64 ops, relative error <= 3e-13) and the
//            decisions are re-run with bounds of ~V*2^-52.
//   EXACT    (separate kernel, queued) emulation of numpy's operation order
//            (pairwise sums, sequential cumsum, lexsort order).  Only the libm
//            exp can differ from numpy's (<= 1 ulp); a draw whose margin is
//            within that is flagged LC_DRAW_UNRESOLVED.
//
// Layout: one CTA (256 threads, 2 CTAs per SM) per task, persistent over
// tasks.  Warp w owns the contiguous id range [w*C, (w+1)*C) of the row (C a
// multiple of 8); a lane reads 8 consecutive elements per 16 B (bf16) / 32 B
// (fp32) vector, so a warp instruction covers 256 consecutive ids (coalesced)
// and warp ranges are in id order -- what the inverse-CDF search needs.
#include <float.h>
#include <limits.h>
#include <math.h>
#include <stdlib.h>

#include "lc_common.cuh"
#include "lc_numpy.cuh"
#include "lc_resample.cuh"
#include "lc_task.cuh"
#include "lc_probs.cuh"

namespace lcb {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_MIN_BLOCKS = 2;      // CTAs per SM (registers <= 128/thread)
constexpr int CAND_CAP = 1024;        // candidate list (top-k / small nucleus / bracket) in smem
constexpr int NBINS = 256;            // nucleus histogram bins
constexpr float BINS_PER_OCT = 4.0f;  // 64 octaves of dynamic range
constexpr int K0_SPEC = 64;           // speculative candidate count for top-p without top-k
constexpr int SCR_PER_WARP = 2048;    // large-nucleus kept elements per warp (global scratch)
constexpr int SCR_PER_CTA = SCR_PER_WARP * RS_WARPS;


// ---- loading --------------------------------------------------------------------------------

// 8 consecutive logits starting at id e0; ids >= lim read as -inf.
template <int DT>
__device__ __forceinline__ void load8(const char* row, int e0, int lim, bool vec, float v[8]) {
  if (e0 >= lim) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = -INFINITY;
    return;
  }
  if (DT == LC_BF16) {
    const uint16_t* r = reinterpret_cast<const uint16_t*>(row);
    if (vec && e0 + 8 <= lim) {
      uint4 q = __ldg(reinterpret_cast<const uint4*>(r + e0));
      uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[2 * j] = __uint_as_float(w[j] << 16);
        v[2 * j + 1] = __uint_as_float(w[j] & 0xffff0000u);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (e0 + j < lim) ? bf16_bits_to_f32(__ldg(r + e0 + j)) : -INFINITY;
    }
  } else {
    const float* r = reinterpret_cast<const float*>(row);
    if (vec && e0 + 8 <= lim) {
      float4 a = __ldg(reinterpret_cast<const float4*>(r + e0));
      float4 b = __ldg(reinterpret_cast<const float4*>(r + e0 + 4));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (e0 + j < lim) ? __ldg(r + e0 + j) : -INFINITY;
    }
  }
}

// Warp-uniform pass over the warp's id range [cb, ce): UNR vectors per lane are
// loaded before any is consumed (memory-level parallelism); f(e0, v) sees ids
// e0..e0+7, ids >= ce read as -inf (callers mask with e0 + j < ce).
template <int DT, int UNR, typename F>
__device__ __forceinline__ void warp_pass(const char* row, int cb, int ce, bool vec, int lane, F&& f) {
  for (int base = cb; base < ce; base += 256 * UNR) {
    float v[UNR][8];
#pragma unroll
    for (int u = 0; u < UNR; ++u) load8<DT>(row, base + 256 * u + 8 * lane, ce, vec, v[u]);
#pragma unroll
    for (int u = 0; u < UNR; ++u) f(base + 256 * u + 8 * lane, v[u]);
  }
}

template <int DT>
__device__ __forceinline__ float load1(const char* row, int i) {
  if (DT == LC_BF16) return bf16_bits_to_f32(__ldg(reinterpret_cast<const uint16_t*>(row) + i));
  return __ldg(reinterpret_cast<const float*>(row) + i);
}


// Phase A: per-thread max and min over the warp's id range, NaN-propagating,
// packed bf16x2 for bf16 rows (one HMNMX2 per two elements).
template <int DT>
__device__ __forceinline__ void phase_a(const char* row, int cb, int ce, bool vec, int lane, float& tmax, float& tmin) {
  if (DT == LC_BF16 && vec) {
    const uint16_t* r = reinterpret_cast<const uint16_t*>(row);
    __nv_bfloat162 mx = __float2bfloat162_rn(-INFINITY), mn = __float2bfloat162_rn(INFINITY);
    for (int base = cb; base < ce; base += 256 * 8) {
      uint4 q[8];
      bool full[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e0 = base + 256 * u + 8 * lane;
        full[u] = e0 + 8 <= ce;
        if (full[u]) q[u] = __ldg(reinterpret_cast<const uint4*>(r + e0));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e0 = base + 256 * u + 8 * lane;
        if (full[u]) {
          const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(&w[k]);
            mx = __hmax2_nan(mx, x);
            mn = __hmin2_nan(mn, x);
          }
        } else {
          for (int j = 0; j < 8 && e0 + j < ce; ++j) {
            const float f = bf16_bits_to_f32(r[e0 + j]);
            tmax = max_nan(tmax, f);
            tmin = min_nan(tmin, f);
          }
        }
      }
    }
    tmax = max_nan(tmax, max_nan(__low2float(mx), __high2float(mx)));
    tmin = min_nan(tmin, min_nan(__low2float(mn), __high2float(mn)));
  } else {
    warp_pass<DT, 4>(row, cb, ce, vec, lane, [&](int e0, const float* v) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        tmax = max_nan(tmax, v[j]);
        if (e0 + j < ce) tmin = min_nan(tmin, v[j]);
      }
    });
  }
}

// Phase A for the row-per-warp kernel: also records, per lane, the first
// vector (id of its first element) holding the lane's maximum, so the first
// argmax costs one reload instead of a scan.
template <int DT>
__device__ __forceinline__ void phase_a_pos(const char* row, int V, bool vec, int lane, float& tmax, float& tmin,
                                            int& tpos) {
  if (DT == LC_BF16 && vec) {
    const uint16_t* r = reinterpret_cast<const uint16_t*>(row);
    for (int base = 0; base < V; base += 256 * 8) {
      uint4 q[8];
      bool full[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e0 = base + 256 * u + 8 * lane;
        full[u] = e0 + 8 <= V;
        if (full[u]) q[u] = __ldg(reinterpret_cast<const uint4*>(r + e0));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e0 = base + 256 * u + 8 * lane;
        float vmax, vmin;
        if (full[u]) {
          const __nv_bfloat162 a0 = *reinterpret_cast<const __nv_bfloat162*>(&q[u].x);
          const __nv_bfloat162 a1 = *reinterpret_cast<const __nv_bfloat162*>(&q[u].y);
          const __nv_bfloat162 a2 = *reinterpret_cast<const __nv_bfloat162*>(&q[u].z);
          const __nv_bfloat162 a3 = *reinterpret_cast<const __nv_bfloat162*>(&q[u].w);
          const __nv_bfloat162 mx = __hmax2_nan(__hmax2_nan(a0, a1), __hmax2_nan(a2, a3));
          const __nv_bfloat162 mn = __hmin2_nan(__hmin2_nan(a0, a1), __hmin2_nan(a2, a3));
          vmax = max_nan(__low2float(mx), __high2float(mx));
          vmin = min_nan(__low2float(mn), __high2float(mn));
        } else {
          vmax = -INFINITY;
          vmin = INFINITY;
          for (int j = 0; j < 8 && e0 + j < V; ++j) {
            const float f = bf16_bits_to_f32(r[e0 + j]);
            vmax = max_nan(vmax, f);
            vmin = min_nan(vmin, f);
          }
        }
        if (vmax > tmax || vmax != vmax) {
          tmax = (vmax != vmax || tmax != tmax) ? NAN : vmax;
          tpos = e0;
        }
        tmin = min_nan(tmin, vmin);
      }
    }
  } else {
    for (int base = 0; base < V; base += 256 * 4) {
      float v[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) load8<DT>(row, base + 256 * u + 8 * lane, V, vec, v[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e0 = base + 256 * u + 8 * lane;
        float vmax = max_nan(max_nan(max_nan(v[u][0], v[u][1]), max_nan(v[u][2], v[u][3])),
                             max_nan(max_nan(v[u][4], v[u][5]), max_nan(v[u][6], v[u][7])));
        float vmin = INFINITY;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (e0 + j < V) vmin = min_nan(vmin, v[u][j]);
        if (vmax > tmax || vmax != vmax) {
          tmax = (vmax != vmax || tmax != tmax) ? NAN : vmax;
          tpos = e0;
        }
        tmin = min_nan(tmin, vmin);
      }
    }
  }
}


// REFINE-grade exp for candidate values: the reference's own argument
// s = fl(fl(z/T) - fl(m/T)), then the fp64 libm exponential (<= 1 ulp).
__device__ __forceinline__ double ref_exp(const ExpCtx& c, float z) {
  double s = __dsub_rn(__ddiv_rn((double)z, c.T), c.mT);
  return exp(s);
}

// 2^(b/4) (fp32, relative error <= 2^-24)
__device__ __forceinline__ float bin_scale(int b) {
  const float frac = (b & 3) == 0 ? 1.0f : (b & 3) == 1 ? 1.18920711500272f : (b & 3) == 2 ? 1.41421356237310f
                                                                                            : 1.68179283050743f;
  return __int_as_float(((b >> 2) + 127) << 23) * frac;
}

// log2-distance bin of z below the max (monotone non-increasing in z)
__device__ __forceinline__ int nbin(const ExpCtx& c, float z) {
  float a = (z - c.m) * c.Lhi;
  return max((int)fminf(-a * BINS_PER_OCT, (float)(NBINS - 1)), 0);
}

// ---- keys ----------------------------------------------------------------------------------

// (z desc, id asc) == numeric descending order of this key
__device__ __forceinline__ unsigned long long cand_key(float z, int id) {
  return ((unsigned long long)f32_order_key(z) << 32) | (unsigned long long)(0xffffffffu - (uint32_t)id);
}
__device__ __forceinline__ int cand_id(unsigned long long k) { return (int)(0xffffffffu - (uint32_t)(k & 0xffffffffu)); }
__device__ __forceinline__ float cand_z(unsigned long long k) {
  uint32_t o = (uint32_t)(k >> 32);
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(u);
}

// ---- shared memory ----------------------------------------------------------------------------

struct __align__(16) Smem {
  unsigned long long cand[CAND_CAP];  // candidate keys
  double ce[CAND_CAP];                // precise e of sorted candidates
  int sl_id[CAND_CAP];                // kept small list, id order
  double sl_e[CAND_CAP];              // its e, later its inclusive prefix
  uint32_t hist[RS_WARPS][NBINS];     // per-warp fixed-point nucleus histogram
  unsigned long long tmp64[RS_THREADS];
  double t16[16];                     // 2^(j/16) for lite_exp
  double wsum[RS_WARPS];
  double werr[RS_WARPS];
  double wpre[RS_WARPS + 1];
  float wmax[RS_WARPS];
  float wmin[RS_WARPS];
  float wtheta[RS_WARPS];
  int warg[RS_WARPS];
  int wcount[RS_WARPS];
  int wsl[RS_WARPS + 1];
  double dsc[4];
  int isc[8];
};
// isc: 0 candidate count, 1 bad row, 2 overflow, 3 kept count, 4 uncertain, 5 blo, 6 bhi, 7 draw uncertain

// Descending bitonic sort of n (power of two) 64-bit keys in smem.
__device__ void bitonic_desc(unsigned long long* a, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += RS_THREADS) {
        int p = i ^ j;
        if (p > i) {
          unsigned long long x = a[i], y = a[p];
          bool desc = ((i & k) == 0);
          if (desc ? (x < y) : (x > y)) {
            a[i] = y;
            a[p] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

// r-th largest (1-based) of the 32 lane values, via a warp bitonic sort.
__device__ __forceinline__ float warp_rth_largest(float v, int r) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      float o = __shfl_xor_sync(0xffffffffu, v, j);
      bool desc = (lane & k) == 0 || k == 32;
      bool lower = (lane & j) == 0;
      v = (lower == desc) ? fmaxf(v, o) : fminf(v, o);
    }
  }
  return __shfl_sync(0xffffffffu, v, r - 1);
}

// Sort n distinct keys descending (n <= CAND_CAP): rank by counting for
// n <= RS_THREADS, bitonic otherwise.
__device__ void sort_desc(unsigned long long* a, int n, unsigned long long* tmp) {
  if (n <= RS_THREADS) {
    unsigned long long k = 0;
    int rank = 0;
    if ((int)threadIdx.x < n) {
      k = a[threadIdx.x];
      for (int j = 0; j < n; ++j) rank += (a[j] > k);
    }
    __syncthreads();
    if ((int)threadIdx.x < n) tmp[rank] = k;
    __syncthreads();
    if ((int)threadIdx.x < n) a[threadIdx.x] = tmp[threadIdx.x];
    __syncthreads();
    return;
  }
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  for (int i = n + threadIdx.x; i < n2; i += RS_THREADS) a[i] = 0ull;
  __syncthreads();
  bitonic_desc(a, n2);
}

// warp-aggregated append to sm.cand
__device__ __forceinline__ void push_cand(Smem& sm, bool pred, float z, int id, int& overflow) {
  unsigned mask = __ballot_sync(0xffffffffu, pred);
  if (mask == 0) return;
  int lane = threadIdx.x & 31;
  int leader = __ffs(mask) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(&sm.isc[0], __popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (pred) {
    int pos = base + __popc(mask & ((1u << lane) - 1u));
    if (pos < CAND_CAP) sm.cand[pos] = cand_key(z, id);
    else overflow = 1;
  }
}

// inclusive warp scan (fp64)
__device__ __forceinline__ double warp_incl_scan(double x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}


// counters: 0 tasks that needed the PRECISE pass, 1 unresolved draws (EXACT),
// 2 bad rows, 3 tasks sent to EXACT, 4 uncertain cut (FAST), 5 uncertain draw
// (FAST), 6 uncertain after PRECISE, 7 candidate/scratch overflow.

// ============================== FAST + PRECISE kernel ==============================

template <int DT>
__global__ void __launch_bounds__(RS_THREADS, RS_MIN_BLOCKS)
resample_kernel(const char* __restrict__ rows, int64_t row_bytes, int Vdef, const lc_task* __restrict__ tasks,
                int n_tasks, CacheMap cm, DrawIO io, Workspace ws, unsigned long long* counters, int rw_owns,
                int force) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem& sm = *reinterpret_cast<Smem*>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* scrA_id = ws.scr_id + (int64_t)blockIdx.x * 2 * SCR_PER_CTA;
  double* scrA_e = ws.scr_e + (int64_t)blockIdx.x * 2 * SCR_PER_CTA;
  int* scrM_id = scrA_id + SCR_PER_CTA;
  double* scrM_e = scrA_e + SCR_PER_CTA;
  if (tid < 16) sm.t16[tid] = exp2((double)tid / 16.0);

  // with the row-warp kernel in front, only the tasks it queued (effective top-k)
  const int n_mine = rw_owns ? *(volatile int*)ws.q_cta : n_tasks;
  for (int qi = blockIdx.x; qi < n_mine; qi += gridDim.x) {
    const int task_id = rw_owns ? ws.q_cta[1 + qi] : qi;
    const lc_task tk = tasks[task_id];
    if (tk.draw_end <= tk.draw_begin) continue;  // nothing to draw (uniform across the CTA)
    TaskView tv;
    __syncthreads();  // previous task's smem readers are done
    if (!resolve_task(tk, rows, row_bytes, Vdef, cm, tv)) {
      write_all(tv, io, -1, LC_DRAW_BAD_ROW);
      if (tid == 0) {
        atomicAdd(&counters[2], 1ull);
        set_kept(io, task_id, -1);
      }
      continue;
    }
    if (force == 2) {  // test hook: everything to the EXACT tier
      if (tid == 0) {
        const int pos = atomicAdd(ws.q_exact, 1);
        ws.q_exact[1 + pos] = task_id;
      }
      continue;
    }
    const int V = tv.V;
    const bool vec = ((reinterpret_cast<uintptr_t>(tv.row) & 15) == 0);
    const int C = ((V + RS_WARPS - 1) / RS_WARPS + 7) & ~7;
    const int cb = min(V, warp * C);
    const int ce = min(V, cb + C);
    if (tid < 8) sm.isc[tid] = 0;

    // ---------------- phase A: max, first argmax, |z| range, thread maxima, NaN check
    float tmax = -INFINITY, tmin = INFINITY;
    phase_a<DT>(tv.row, cb, ce, vec, lane, tmax, tmin);
    const bool bad = (tmax != tmax) || (tmin != tmin);
    if (bad) tmax = -INFINITY;
    __syncthreads();  // isc reset visible
    {
      float wm = warp_max(tmax);
      float wn = -warp_max(-tmin);
      bool wbad = __any_sync(0xffffffffu, bad);
      if (lane == 0) {
        sm.wmax[warp] = wm;
        sm.wmin[warp] = wn;
        if (wbad) sm.isc[1] = 1;
      }
    }
    __syncthreads();
    float m = -INFINITY, zmin = INFINITY;
    for (int w = 0; w < RS_WARPS; ++w) {
      m = fmaxf(m, sm.wmax[w]);
      zmin = fminf(zmin, sm.wmin[w]);
    }
    const uint8_t base_flag = 0;
    if (sm.isc[1] || !(m > -INFINITY) || !(m < INFINITY)) {
      write_all(tv, io, -1, LC_DRAW_BAD_ROW);
      if (tid == 0) {
        atomicAdd(&counters[2], 1ull);
        set_kept(io, task_id, -1);
      }
      continue;
    }
    // first argmax (lowest id with z == m), computed lazily: greedy rows need it now
    auto first_argmax = [&]() -> int {
      int best = INT_MAX;
      warp_pass<DT, 2>(tv.row, cb, ce, vec, lane, [&](int e0, const float* v) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (v[j] == m && e0 + j < best) best = e0 + j;
      });
      best = warp_min_int(best);
      __syncthreads();
      if (lane == 0) sm.warg[warp] = best;
      __syncthreads();
      int a = INT_MAX;
      for (int w = 0; w < RS_WARPS; ++w) a = min(a, sm.warg[w]);
      return a;
    };
    if (tv.T == 0.0) {  // greedy: one-hot at the first argmax, still one draw (sampling.py:61-64)
      const int amax = first_argmax();
      write_all(tv, io, amax, base_flag);
      if (tid == 0) set_kept(io, task_id, greedy_kept(V, tv.topk, tv.topp));
      continue;
    }
    ExpCtx ec;
    ec.m = m;
    ec.T = tv.T;
    ec.mT = __ddiv_rn((double)m, tv.T);
    ec.md = (double)m;
    {
      double Ld = 1.4426950408889634 / tv.T;
      ec.Lhi = (float)Ld;
      ec.Llo = (float)(Ld - (double)ec.Lhi);
      ec.L16 = 16.0 * Ld;
    }
    // temperatures whose scaled logits leave the fp32 / table range go to EXACT
    const double zabs = fmax(fabs((double)m), isfinite(zmin) ? fabs((double)zmin) : fabs((double)m));
    const bool sane = ec.Lhi < 1e20f && ec.Lhi > 1e-20f && fabsf(m) * ec.Lhi < 1e30f && zabs / tv.T < 1e15;
    // reference argument rounding: |s_ref - s| <= 2^-51 (|z| + |m|) / T  (relative error of e)
    const double relArg = 4.440892098500626e-16 * 2.0 * zabs / tv.T;
    const double relRef = (double)(2 * V + 64) * kEps64;  // reference's rounding of p, csum, sum(q), cumsum

    // ---------------- candidate threshold (top-k, or speculative small nucleus)
    int kc = 0;
    if (tv.topk > 0) kc = tv.topk;
    else if (tv.trunc && tv.topp < 1.0) kc = K0_SPEC;
    float theta = INFINITY;
    if (kc > 0 && kc <= 32 * RS_WARPS) {
      // every warp has r = ceil(kc/WARPS) thread maxima >= its r-th largest, so
      // the minimum over warps lower-bounds the kc-th largest logit
      const int r = (kc + RS_WARPS - 1) / RS_WARPS;
      float tw = warp_rth_largest(tmax, r);
      if (lane == 0) sm.wtheta[warp] = tw;
      __syncthreads();
      for (int w = 0; w < RS_WARPS; ++w) theta = fminf(theta, sm.wtheta[w]);
    } else if (kc > 0) {
      theta = -INFINITY;  // collect all; overflow -> EXACT
    }

    // ---------------- phase B: fast mass per warp, candidates
    // truncated rows only need the mass for the nucleus target (bound via W);
    // untruncated rows need tight per-element errors for the draw itself
    const bool accurate = !tv.trunc;
    double S_part = 0.0;
    float W_part = 0.0f;
    int overflow = 0;
    auto push_lane = [&](unsigned m8, int e0, const float* v) {
      const int cnt = __popc(m8);
      if (__any_sync(0xffffffffu, cnt != 0)) {
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        int base = 0;
        if (lane == 31) base = atomicAdd(&sm.isc[0], incl);
        base = __shfl_sync(0xffffffffu, base, 31);
        int pos = base + incl - cnt;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if ((m8 >> j) & 1u) {
            if (pos < CAND_CAP) sm.cand[pos] = cand_key(v[j], e0 + j);
            else overflow = 1;
            ++pos;
          }
        }
      }
    };
    if (accurate) {
      warp_pass<DT, 2>(tv.row, cb, ce, vec, lane, [&](int e0, const float* v) {
        float e[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) e[j] = fast_exp(ec, v[j]);  // ids >= ce are -inf -> 0
        S_part += (double)(((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7])));
      });
    } else {
      warp_pass<DT, 2>(tv.row, cb, ce, vec, lane, [&](int e0, const float* v) {
        float e[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float a;
          e[j] = cheap_exp(ec, v[j], a);
          W_part = fmaf(e[j], -a, W_part);
        }
        S_part += (double)(((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7])));
        if (kc > 0) {
          unsigned m8 = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) m8 |= (unsigned)((e0 + j < ce) && v[j] >= theta) << j;
          push_lane(m8, e0, v);
        }
      });
    }
    {
      double wsm = warp_sum(S_part);
      double wW = warp_sum((double)W_part);
      int wo = __any_sync(0xffffffffu, overflow);
      if (lane == 0) {
        sm.wsum[warp] = wsm;
        sm.werr[warp] = wW;
        if (wo) sm.isc[2] = 1;
      }
    }
    __syncthreads();
    const int ncand = min(sm.isc[0], CAND_CAP);
    const bool cand_ok = (sm.isc[2] == 0) && kc > 0 && ncand >= kc;
    double Wrow = 0.0;
    for (int w = 0; w < RS_WARPS; ++w) Wrow += sm.werr[w];
    Wrow *= 1.001;  // fp32 accumulation of a bound quantity
    // first argmax: lowest id among candidates with z == m (the candidates hold every z >= theta <= m)
    int amax = INT_MAX;
    if (cand_ok) {
      int best = INT_MAX;
      for (int i = tid; i < ncand; i += RS_THREADS)
        if (cand_z(sm.cand[i]) == m) best = min(best, cand_id(sm.cand[i]));
      best = warp_min_int(best);
      if (lane == 0) sm.warg[warp] = best;
      __syncthreads();
      for (int w = 0; w < RS_WARPS; ++w) amax = min(amax, sm.warg[w]);
    }
    __syncthreads();

    // per-row state kept across the FAST and PRECISE decision passes
    bool cands_sorted = false;   // small list sorted + ce computed
    int large_state = 0;         // 0 not built, 1 built, -1 failed
    bool to_exact = !sane;
    bool done = false;

    for (int pass = force == 1 ? 1 : 0; pass < 2 && !done && !to_exact; ++pass) {
      const bool precise = pass == 1;
      const uint8_t tier_flag = precise ? LC_DRAW_PRECISE : 0;
      if (precise) {
        // ---- PRECISE: recompute per-warp masses with lite_exp (fp64)
        if (tid == 0) atomicAdd(&counters[0], 1ull);
        double acc = 0.0;
        warp_pass<DT, 2>(tv.row, cb, ce, vec, lane, [&](int e0, const float* v) {
#pragma unroll
          for (int j = 0; j < 8; ++j) acc += lite_exp(ec, v[j], sm.t16);
        });
        acc = warp_sum(acc);
        __syncthreads();
        if (lane == 0) sm.wsum[warp] = acc;
        __syncthreads();
      }
      double S = 0.0;
      for (int w = 0; w < RS_WARPS; ++w) S += sm.wsum[w];
      const double relE = precise    ? (kLiteErr + 2.0 * kRefExpErr + relArg + (double)(V + 16) * kEps64)
                          : accurate ? (kEx2RelErr + kCorrErr + kSum8Err + kRefExpErr + relArg +
                                        (double)(V + 16) * kEps64)
                                     : (kEx2Raw + kSum8Err + kRefExpErr + relArg + (double)(V + 16) * kEps64);
      const double absE = precise ? (double)V * 1e-300 : (double)V * 2.4e-38;  // flushed / subnormal mass
      const double E_S = S * relE + absE + ((!precise && !accurate) ? kArgRel * Wrow : 0.0);
      bool unc = false;

      // Kept-set representation for the draw:
      //   mode 0 -- untruncated: all ids, e recomputed by the owning warp;
      //   mode 1 -- small list sl_id/sl_e (id order) of length L;
      //   mode 2 -- per-warp merged lists in global scratch (scrM), counts wcount[].
      int mode = 0;
      int L = 0;

      if (tv.trunc && tv.topp < 1.0) {
        // p(first argmax) = 1/S (its e is exactly 1 in both implementations); if it
        // certainly reaches top_p the nucleus is {argmax} and every draw returns it
        const double pmax_lo = (1.0 / (S + E_S)) * (1.0 - relRef);
        if (pmax_lo > tv.topp) {
          if (amax == INT_MAX) amax = first_argmax();
          write_all(tv, io, amax, tier_flag);
          if (tid == 0) set_kept(io, task_id, 1);
          done = true;
          break;
        }
      }

      if (tv.trunc) {
        const double P = tv.topp * S;  // nucleus target in e-space
        bool small_done = false;
        if (cand_ok && large_state == 0) {
          if (!cands_sorted) {
            sort_desc(sm.cand, ncand, sm.tmp64);
            const int klim0 = tv.topk > 0 ? tv.topk : ncand;
            for (int i = tid; i < klim0; i += RS_THREADS) sm.ce[i] = ref_exp(ec, cand_z(sm.cand[i]));
            __syncthreads();
            cands_sorted = true;
          }
          const int klim = tv.topk > 0 ? tv.topk : ncand;
          if (warp == 0) {
            // inclusive scan of the sorted candidates' e; first crossing of P
            int cut = -1;
            bool u_ = false;
            if (tv.topp < 1.0) {
              double off = 0.0;
              for (int i0 = 0; i0 < klim; i0 += 32) {
                const int i = i0 + lane;
                const double e = i < klim ? sm.ce[i] : 0.0;
                const double c = off + warp_incl_scan(e), prev = c - e;
                const double tol = tv.topp * E_S + c * relRef;
                const unsigned hm = __ballot_sync(0xffffffffu, i < klim && c >= P - tol);
                if (hm) {
                  const int hl = __ffs(hm) - 1;
                  cut = i0 + hl;
                  const bool ok = (c - P > tol && P - prev > tol);
                  u_ = !__shfl_sync(0xffffffffu, ok, hl);
                  break;
                }
                off = __shfl_sync(0xffffffffu, c, 31);
              }
            }
            int Lk = cut >= 0 ? cut + 1 : (tv.topk > 0 ? klim : -1);
            if (Lk > 0) {
              // distinct logits that the reference might round to equal p: ordering unsafe
              const int lim = min(Lk + 1, ncand);
              bool bad_order = false;
              for (int i = 1 + lane; i < lim; i += 32) {
                float za = cand_z(sm.cand[i - 1]), zb = cand_z(sm.cand[i]);
                if (za != zb) {
                  double da = __ddiv_rn((double)za, tv.T), db = __ddiv_rn((double)zb, tv.T);
                  if (da - db <= fmax(fabs(da), fabs(ec.mT)) * 8.0 * kEps64) bad_order = true;
                }
              }
              u_ |= __any_sync(0xffffffffu, bad_order);
            }
            if (lane == 0) {
              sm.isc[3] = Lk;
              sm.isc[4] = u_;
            }
          }
          __syncthreads();
          const int Lk = sm.isc[3];
          if (sm.isc[4]) unc = true;
          else if (Lk > 0) {
            small_done = true;
            mode = 1;
            L = Lk;
          }
          __syncthreads();
        } else if (tv.topk > 0) {
          to_exact = true;  // top-k candidates overflowed (heavy ties / k > 256) -> EXACT
          if (tid == 0) atomicAdd(&counters[7], 1ull);
          break;
        }

        if (!unc && !small_done) {
          // -------- large nucleus: top-p without top-k, nucleus beyond the speculative list
          if (large_state == 0) {
            for (int i = tid; i < RS_WARPS * NBINS; i += RS_THREADS) (&sm.hist[0][0])[i] = 0u;
            __syncthreads();
            // per-bin relative fixed point: bin b holds e in (2^-(b+1)/4, 2^-b/4] (up to the
            // approximate binning argument), so q = e * 2^(b/4) * qscale is < 2^31/C per element
            // and the bin mass carries a relative error <= 2^-(31-lgC)/0.8 + fast_exp's.
            const int lgC = 32 - __clz(C + 1);
            const float qscale = ldexpf(1.0f, 30 - lgC);
            warp_pass<DT, 2>(tv.row, cb, ce, vec, lane, [&](int e0, const float* v) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (e0 + j < ce) {
                  const int b = nbin(ec, v[j]);
                  float a;
                  const float q = cheap_exp(ec, v[j], a) * bin_scale(b) * qscale;
                  atomicAdd(&sm.hist[warp][b], __float2uint_rn(fminf(q, 2.0f * qscale)));
                }
            });
            __syncthreads();
            if (warp == 0) {
              // bracket [blo, bhi] of bins that can hold the cut (fast mass + quantisation error)
              const double inv = 1.0 / (double)qscale;
              // quantisation + cheap_exp (|a| <= 64 below the catch-all bin) + bin_scale rounding
              const double qrel = ldexp(1.0, lgC - 30) * 1.25 + kEx2Raw + kArgRel * 64.0 + 1e-7;
              const double qerr = qrel * S + 2.0 * E_S + P * relRef;
              double cum = 0.0;
              int blo = NBINS - 1, bhi = NBINS - 1;
              bool got_lo = false;
              for (int b0 = 0; b0 < NBINS; b0 += 32) {
                unsigned long long hs = 0;
                for (int w = 0; w < RS_WARPS; ++w) hs += sm.hist[w][b0 + lane];
                const double incl = cum + warp_incl_scan((double)hs * inv * exp2(-0.25 * (double)(b0 + lane)));
                const unsigned lo_m = __ballot_sync(0xffffffffu, incl >= P - qerr);
                const unsigned hi_m = __ballot_sync(0xffffffffu, incl >= P + qerr);
                if (!got_lo && lo_m) {
                  blo = b0 + __ffs(lo_m) - 1;
                  got_lo = true;
                }
                if (hi_m) {
                  bhi = b0 + __ffs(hi_m) - 1;
                  break;
                }
                cum = __shfl_sync(0xffffffffu, incl, 31);
              }
              if (lane == 0) {
                sm.isc[5] = blo;
                sm.isc[6] = bhi;
                sm.isc[0] = 0;
                sm.isc[2] = 0;
              }
            }
            __syncthreads();
            const int blo = sm.isc[5], bhi = sm.isc[6];
            // order-preserving per-warp compaction of bins < blo (certainly kept) to
            // scratch A; bracket bins [blo, bhi] to the smem candidate list
            int wn = 0, ovf = 0;
            warp_pass<DT, 2>(tv.row, cb, ce, vec, lane, [&](int e0, const float* v) {
              int b[8];
              int mine = 0;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                b[j] = (e0 + j < ce) ? nbin(ec, v[j]) : NBINS;
                mine += (b[j] < blo);
              }
              const int x = (int)warp_incl_scan((double)mine);
              int pos = wn + x - mine;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                if (b[j] < blo) {
                  if (pos < SCR_PER_WARP) scrA_id[warp * SCR_PER_WARP + pos] = e0 + j;
                  else ovf = 1;
                  ++pos;
                }
              }
              wn += __shfl_sync(0xffffffffu, x, 31);
              unsigned m8 = 0;
#pragma unroll
              for (int j = 0; j < 8; ++j) m8 |= (unsigned)(b[j] >= blo && b[j] <= bhi) << j;
              if (__any_sync(0xffffffffu, m8 != 0)) {
#pragma unroll
                for (int j = 0; j < 8; ++j) push_cand(sm, (m8 >> j) & 1u, v[j], e0 + j, ovf);
              }
            });
            ovf = __any_sync(0xffffffffu, ovf);
            if (lane == 0) {
              sm.wcount[warp] = min(wn, SCR_PER_WARP);
              if (ovf || wn > SCR_PER_WARP) sm.isc[2] = 1;
            }
            __syncthreads();
            if (sm.isc[2]) {
              large_state = -1;
            } else {
              // precise e of the certainly-kept elements (dense, per warp)
              const int nw = sm.wcount[warp];
              double acc = 0.0;
              for (int i = lane; i < nw; i += 32) {
                double e = lite_exp(ec, load1<DT>(tv.row, scrA_id[warp * SCR_PER_WARP + i]), sm.t16);
                scrA_e[warp * SCR_PER_WARP + i] = e;
                acc += e;
              }
              acc = warp_sum(acc);
              if (lane == 0) sm.werr[warp] = acc;  // kept mass above the bracket, per warp
              sort_desc(sm.cand, min(sm.isc[0], CAND_CAP), sm.tmp64);
              const int nb = min(sm.isc[0], CAND_CAP);
              for (int i = tid; i < nb; i += RS_THREADS) sm.ce[i] = ref_exp(ec, cand_z(sm.cand[i]));
              __syncthreads();
              double Mab = 0.0;
              for (int w = 0; w < RS_WARPS; ++w) Mab += sm.werr[w];
              if (tid == 0) sm.dsc[1] = Mab;
              large_state = 1;
            }
            __syncthreads();
          }
          if (large_state < 0) {
            to_exact = true;
            if (tid == 0) atomicAdd(&counters[7], 1ull);
            break;
          }
          const int nb = min(sm.isc[0], CAND_CAP);
          if (warp == 0) {
            const double Mabove = sm.dsc[1];
            const double tolS = tv.topp * E_S + Mabove * (kLiteErr + relArg + 2.0 * kRefExpErr);
            int cut = -1;
            bool u_ = Mabove >= P - tolS - Mabove * relRef;  // the cut would lie above the bracket
            double off = Mabove;
            for (int i0 = 0; i0 < nb && !u_; i0 += 32) {
              const int i = i0 + lane;
              const double e = i < nb ? sm.ce[i] : 0.0;
              const double c = off + warp_incl_scan(e), prev = c - e;
              const double tol = tolS + c * relRef;
              const unsigned hm = __ballot_sync(0xffffffffu, i < nb && c >= P - tol);
              if (hm) {
                const int hl = __ffs(hm) - 1;
                cut = i0 + hl;
                const bool ok = (c - P > tol && P - prev > tol);
                u_ = !__shfl_sync(0xffffffffu, ok, hl);
                break;
              }
              off = __shfl_sync(0xffffffffu, c, 31);
            }
            if (cut < 0) u_ = true;
            if (!u_) {
              bool bad_order = false;
              for (int i = max(cut, 1) + lane; i <= min(cut + 1, nb - 1); i += 32) {
                float za = cand_z(sm.cand[i - 1]), zb = cand_z(sm.cand[i]);
                if (za != zb) {
                  double da = __ddiv_rn((double)za, tv.T), db = __ddiv_rn((double)zb, tv.T);
                  if (da - db <= fmax(fabs(da), fabs(ec.mT)) * 8.0 * kEps64) bad_order = true;
                }
              }
              u_ |= __any_sync(0xffffffffu, bad_order);
            }
            if (lane == 0) {
              sm.isc[3] = cut + 1;
              sm.isc[4] = u_;
            }
          }
          __syncthreads();
          if (sm.isc[4]) {
            unc = true;
          } else {
            mode = 2;
            L = sm.isc[3];  // the first L bracket candidates are kept
          }
          __syncthreads();
        }
        if (unc) {
          if (tid == 0 && !precise) atomicAdd(&counters[4], 1ull);
          continue;  // -> PRECISE pass (or EXACT after it)
        }
      }

      // ---------------- kept small list in id order (modes 1 and 2)
      if (mode != 0) {
        // ids are distinct: rank by counting (L is a top-k, a small nucleus or a bracket prefix)
        for (int i = tid; i < L; i += RS_THREADS) {
          const int id = cand_id(sm.cand[i]);
          int rank = 0;
          for (int j = 0; j < L; ++j) rank += (cand_id(sm.cand[j]) < id);
          sm.sl_id[rank] = id;
          sm.sl_e[rank] = sm.ce[i];
        }
        __syncthreads();
      }

      if (mode == 1) {
        if (warp == 0) {  // inclusive prefix of the kept e's in id order
          double off = 0.0;
          for (int i0 = 0; i0 < L; i0 += 32) {
            const int i = i0 + lane;
            const double e = i < L ? sm.sl_e[i] : 0.0;
            const double c = off + warp_incl_scan(e);
            if (i < L) sm.sl_e[i] = c;
            off = __shfl_sync(0xffffffffu, c, 31);
          }
          if (lane == 0) sm.dsc[0] = off;
        }
        __syncthreads();
        const double K = sm.dsc[0];
        // kept e's are precise: only the reference's rounding and ours remain
        const double tolK = K * ((double)(V + L + 64) * 4.0 * kEps64 + 4.0 * kRefExpErr + 2.0 * relArg);
        int need = 0;
        for (int64_t d = tv.d0 + tid; d < tv.d1; d += RS_THREADS) {
          const double u = draw_u(io, d, tv);
          const double t = u * K;
          int lo = 0, hi = L;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sm.sl_e[mid] > t) hi = mid;
            else lo = mid + 1;
          }
          // lower boundary 0 (nothing kept before) is exact in both implementations
          const bool ok = lo < L && (lo == 0 || t - sm.sl_e[lo - 1] > tolK) && (sm.sl_e[lo] - t > tolK);
          io.token[d] = sm.sl_id[min(lo, L - 1)];
          if (io.flags) io.flags[d] = tier_flag;
          need |= !ok;
        }
        need = __syncthreads_or(need);
        if (!need) {
          done = true;
          if (tid == 0) set_kept(io, task_id, L);  // the first L of the (z desc, id asc) order
        } else if (tid == 0 && !precise) {
          atomicAdd(&counters[5], 1ull);
        }
        continue;
      }

      // ---------------- modes 0 and 2: per-warp masses, the owner warp searches its range
      if (mode == 2) {
        // merge the warp's scratch list A with its kept bracket members into scratch M
        // (both id-ordered): new position = own index + #other-list ids below.
        if (tid <= RS_WARPS) {
          const int w = tid, bound = min(V, w * C);
          int lo = 0, hi = L;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sm.sl_id[mid] < bound) lo = mid + 1;
            else hi = mid;
          }
          sm.wsl[w] = (w == RS_WARPS) ? L : lo;
        }
        __syncthreads();
        const int na = sm.wcount[warp];
        const int s0 = sm.wsl[warp], s1 = sm.wsl[warp + 1];
        if (na + (s1 - s0) > SCR_PER_WARP) {
          if (lane == 0) sm.isc[2] = 1;
        } else {
          for (int i = lane; i < na; i += 32) {
            const int id = scrA_id[warp * SCR_PER_WARP + i];
            int lo = s0, hi = s1;
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (sm.sl_id[mid] < id) lo = mid + 1;
              else hi = mid;
            }
            scrM_id[warp * SCR_PER_WARP + i + (lo - s0)] = id;
            scrM_e[warp * SCR_PER_WARP + i + (lo - s0)] = scrA_e[warp * SCR_PER_WARP + i];
          }
          double add = 0.0;
          for (int b = s0 + lane; b < s1; b += 32) {
            const int id = sm.sl_id[b];
            int lo = 0, hi = na;
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (scrA_id[warp * SCR_PER_WARP + mid] < id) lo = mid + 1;
              else hi = mid;
            }
            scrM_id[warp * SCR_PER_WARP + (b - s0) + lo] = id;
            scrM_e[warp * SCR_PER_WARP + (b - s0) + lo] = sm.sl_e[b];
            add += sm.sl_e[b];
          }
          add = warp_sum(add);
          __syncwarp();  // every lane read sm.wcount[warp] above before lane 0 rewrites it
          if (lane == 0) {
            sm.wsum[warp] = sm.werr[warp] + add;  // kept mass of this warp's range (precise e's)
            sm.wcount[warp] = na + (s1 - s0);
          }
        }
        __syncthreads();
        if (sm.isc[2]) {
          to_exact = true;
          if (tid == 0) atomicAdd(&counters[7], 1ull);
          break;
        }
      }
      int Kc = V;  // mode 0 (untruncated or top_p == 1 without an effective top-k): identity
      if (mode == 2) {
        Kc = 0;  // warp-range lists above the bracket + the kept bracket members
        for (int w = 0; w < RS_WARPS; ++w) Kc += sm.wcount[w];
      }
      if (tid == 0) {
        double c = 0.0;
        for (int w = 0; w < RS_WARPS; ++w) {
          sm.wpre[w] = c;
          c += sm.wsum[w];
        }
        sm.wpre[RS_WARPS] = c;
      }
      __syncthreads();
      const double K = sm.wpre[RS_WARPS];
      // mode 0: per-element relative bound relE on every partial sum (fast or precise e's);
      // mode 2: kept e's are precise
      const double relD = (mode == 0) ? relE
                                      : ((double)(V + 64) * 4.0 * kEps64 + 4.0 * kRefExpErr + 2.0 * relArg + kLiteErr);
      const double absD = (mode == 0) ? absE : 0.0;
      const bool exact_zero_left = precise || mode == 2;  // no flushed mass can precede
      int need = 0;
      for (int64_t dbase = tv.d0; dbase < tv.d1; dbase += 32) {
        const int64_t d = dbase + lane;
        double t = 0.0, u = 0.0;
        bool mine = false;
        if (d < tv.d1) {
          u = draw_u(io, d, tv);
          t = u * K;
          if (!(t < K)) {
            if (warp == 0) need = 1;  // clamp region: let EXACT emulate it
          } else {
            mine = (t >= sm.wpre[warp]) && (t < sm.wpre[warp + 1]);
          }
        }
        const unsigned own = __ballot_sync(0xffffffffu, mine);
        if (!own) continue;
        // the warp's targets, sorted ascending (warp bitonic on (t, lane)), searched in ONE
        // pass over its id range
        const int nown = __popc(own);
        double st = mine ? t : INFINITY;
        int ssrc = lane;
#pragma unroll
        for (int k2 = 2; k2 <= 32; k2 <<= 1) {
#pragma unroll
          for (int j2 = k2 >> 1; j2 > 0; j2 >>= 1) {
            const double ot = __shfl_xor_sync(0xffffffffu, st, j2);
            const int os = __shfl_xor_sync(0xffffffffu, ssrc, j2);
            const bool asc = (lane & k2) == 0 || k2 == 32;
            const bool lower = (lane & j2) == 0;
            const bool take_other = (lower == asc) ? (ot < st || (ot == st && os < ssrc))
                                                   : (ot > st || (ot == st && os > ssrc));
            if (take_other) {
              st = ot;
              ssrc = os;
            }
          }
        }
        const double su = __shfl_sync(0xffffffffu, u, ssrc);  // u of the target held by this lane
        int k = 0;
        double off = sm.wpre[warp];
        // certify + write target k (found/flo/fhi broadcast to all lanes)
        // gm: the hit group's mass when the walk's group sums are fp32 trees (FAST mode 0): the
        // elements inside it are walked in fp64, which differs from that tree by <= kSum8Err gm
        auto finish = [&](int found, double flo, double fhi, double gm = 0.0) {
          const double tt = __shfl_sync(0xffffffffu, st, k);
          const double uu = __shfl_sync(0xffffffffu, su, k);
          const int src = __shfl_sync(0xffffffffu, ssrc, k);
          if (lane == 0) {
            // correlated bound: err(u*K - A) <= rel * ((1-u)*A + u*(K - A)) + abs
            const double tlo = relD * ((1.0 - uu) * flo + uu * (K - flo)) + absD + tt * relRef * 4.0 +
                               kSum8Err * gm;
            const double thi = relD * ((1.0 - uu) * fhi + uu * (K - fhi)) + absD + tt * relRef * 4.0 +
                               kSum8Err * gm;
            const bool ok = found >= 0 && (tt - flo > tlo || (exact_zero_left && flo == 0.0)) && (fhi - tt > thi);
            io.token[dbase + src] = found;
            if (io.flags) io.flags[dbase + src] = tier_flag;
            need |= !ok;
          }
          ++k;
        };
        if (mode == 0) {
          for (int e0 = cb; e0 < ce && k < nown; e0 += 256) {
            const int my0 = e0 + 8 * lane;
            float v[8];
            load8<DT>(tv.row, my0, ce, vec, v);
            double ev[8];
            double ls = 0.0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              ev[j] = precise ? lite_exp(ec, v[j], sm.t16) : (double)fast_exp(ec, v[j]);
              ls += ev[j];
            }
            if (!precise) {
              // the FAST mass pass summed each group of 8 as an fp32 tree: the walk's group sums
              // must be the same numbers, or the walked prefix and the warp-range prefix / K
              // (from that pass) differ by up to kSum8Err x the walked mass -- an error the
              // correlated bound does not cover (cf. the row-warp fix, round 2)
              float f[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) f[j] = (float)ev[j];
              ls = (double)(((f[0] + f[1]) + (f[2] + f[3])) + ((f[4] + f[5]) + (f[6] + f[7])));
            }
            const double x = warp_incl_scan(ls);
            const double tot = __shfl_sync(0xffffffffu, x, 31);
            while (k < nown) {
              const double tk = __shfl_sync(0xffffffffu, st, k);
              if (!(tk < off + tot)) break;
              const unsigned hm = __ballot_sync(0xffffffffu, (ls > 0.0) && (tk < off + x));
              int found = -1;
              double flo = 0.0, fhi = 0.0, gm = 0.0;
              if (hm) {
                const int hl = __ffs(hm) - 1;
                if (lane == hl) {
                  double c = off + (x - ls);
                  for (int j = 0; j < 8; ++j) {
                    const double nc = c + ev[j];
                    if (ev[j] > 0.0 && tk < nc) {
                      found = my0 + j;
                      flo = c;
                      fhi = nc;
                      break;
                    }
                    c = nc;
                  }
                }
                found = __shfl_sync(0xffffffffu, found, hl);
                flo = __shfl_sync(0xffffffffu, flo, hl);
                fhi = __shfl_sync(0xffffffffu, fhi, hl);
                gm = precise ? 0.0 : __shfl_sync(0xffffffffu, ls, hl);
              }
              finish(found, flo, fhi, gm);
            }
            off += tot;
          }
        } else {
          const int n = sm.wcount[warp];
          for (int i0 = 0; i0 < n && k < nown; i0 += 32) {
            const int i = i0 + lane;
            double e = 0.0;
            int id = -1;
            if (i < n) {
              e = scrM_e[warp * SCR_PER_WARP + i];
              id = scrM_id[warp * SCR_PER_WARP + i];
            }
            const double x = warp_incl_scan(e);
            const double tot = __shfl_sync(0xffffffffu, x, 31);
            while (k < nown) {
              const double tk = __shfl_sync(0xffffffffu, st, k);
              if (!(tk < off + tot)) break;
              const unsigned hm = __ballot_sync(0xffffffffu, (i < n) && (e > 0.0) && (tk < off + x));
              int found = -1;
              double flo = 0.0, fhi = 0.0;
              if (hm) {
                const int hl = __ffs(hm) - 1;
                found = __shfl_sync(0xffffffffu, id, hl);
                flo = __shfl_sync(0xffffffffu, off + x - e, hl);
                fhi = __shfl_sync(0xffffffffu, off + x, hl);
              }
              finish(found, flo, fhi);
            }
            off += tot;
          }
        }
        while (k < nown) finish(-1, 0.0, 0.0);  // rounding left a target past the range end
      }
      need = __syncthreads_or(need);
      if (!need) {
        done = true;
        if (tid == 0) set_kept(io, task_id, Kc);
      } else if (tid == 0 && !precise) {
        atomicAdd(&counters[5], 1ull);
      }
    }

    if (!done) {
      // FAST and PRECISE could not certify (or row too extreme): numpy emulation
      if (tid == 0) {
        int pos = atomicAdd(ws.q_exact, 1);
        ws.q_exact[1 + pos] = task_id;
        atomicAdd(&counters[3], 1ull);
      }
    }
  }
}

// ============================== row-per-warp kernel ==============================
//
// The headline regime (BASELINE configs 1 and 2): many rows, V <= 65536, no
// top-k.  One warp owns one task at a time -- no block barriers, per-warp
// shared state, 24 warps per SM.  Lane l reads the 8-element vectors
// l, l+32, ... so a warp instruction covers 256 consecutive ids; the row is
// cut into 2048-id segments whose masses give the inverse-CDF search a prefix
// table (a draw rescans one segment).
//
// Nucleus without top-k: the first argmax alone (fast exit), or a "big"
// nucleus located by a per-warp fixed-point histogram (8 bins per octave of
// distance from the max), whose bracket bins are sorted exactly; the kept mass
// above the bracket is accumulated per segment in the same pass, so no kept
// list is materialised -- a draw rescans its segment with the kept predicate.
// Tasks with an effective top-k are left to the CTA kernel.

constexpr int RW_THREADS = 256;
constexpr int RW_WARPS = RW_THREADS / 32;
constexpr int RW_MIN_BLOCKS = 2;
constexpr int RW_CAND = 256;      // bracket candidates per warp
constexpr int RW_NB = 1024;       // histogram bins: 32 per octave over 32 octaves (+ catch-all)
constexpr float RW_BPO = 32.0f;
constexpr int RW_SEGSTEPS = 8;    // 8 x 256 ids = 2048 per segment
#ifndef LCB_RW_PF
#define LCB_RW_PF 0  // segments prefetched into L2 ahead of the fused pass (2: +0.3%, 4: -5%; off)
#endif
constexpr int RW_SEG = 256 * RW_SEGSTEPS;
constexpr int RW_MAXV = 65536;
constexpr int RW_NSEG = RW_MAXV / RW_SEG;  // 32
constexpr int RW_NCH = 256;                // kept-list chunks of 32 entries per warp

struct __align__(16) RwWarp {
  unsigned long long cand[RW_CAND];
  double ce[RW_CAND];
  union {
    uint32_t hist[RW_NB];  // big nucleus: histogram (dead once the bracket is known)
    struct {
      double chunk_above[RW_NCH];    // kept list: per-32-entry mass above the bracket
      double chunk_tot[RW_NCH + 1];  // kept list: per-chunk kept mass, then exclusive prefix
    };
  };
  double seg[RW_NSEG + 1];  // segment masses, then exclusive prefix
  double segE[RW_NSEG];     // fused pass: per-segment absolute error bound
  float segm[RW_NSEG];      // fused pass: the warp's running max at the segment end
  double dsc[4];
  int isc[4];
};

struct __align__(16) RwSmem {
  RwWarp w[RW_WARPS];
  double t16[16];
};

__device__ __forceinline__ int rw_bin(float a) {
  // a = log2 distance below the max (<= 0)
  return min((int)(-a * RW_BPO), RW_NB - 1);
}

// the histogram's bin of z: monotone non-increasing in z
__device__ __forceinline__ int rw_zbin(const ExpCtx& c, float z) {
  return rw_bin(fmaxf((z - c.m) * c.Lhi, -200.0f));
}

// smallest z with rw_zbin(z) <= B, for 0 <= B < RW_NB - 1 (bisection over the
// ordered fp32 keys; rw_zbin(m) = 0, rw_zbin(-inf) = RW_NB - 1); +inf for B < 0
__device__ __forceinline__ float rw_zthr(const ExpCtx& c, int B) {
  if (B < 0) return INFINITY;
  auto key2f = [](uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k); };
  uint32_t lo = f32_order_key(-INFINITY), hi = f32_order_key(c.m);
  while (hi - lo > 1u) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    if (rw_zbin(c, key2f(mid)) <= B) hi = mid;
    else lo = mid;
  }
  return key2f(hi);
}

struct FusedOut {
  float tmax, tmin;
  int tpos;
  bool nan;
  double S, ES, relmax;
};

// FAST fused pass (phase A + B in one read): per lane a running maximum mt; the
// lane's partial mass is kept relative to mt and rescaled (factor f with its
// own error bound) when mt grows; at each 2048-id segment end the lanes combine
// at the warp's running max, and at the end every segment is rescaled (fp64)
// to the row max.  Returns the row mass S, its absolute error bound ES and the
// largest per-segment relative bound (for prefix sums), with seg[] relative to
// the row max.  ACC selects the corrected exponential (untruncated rows).
template <int DT, bool ACC>
__device__ __noinline__ FusedOut rw_fused_pass(const char* row, int V, int nseg, bool vec, int lane, float Lhi, float Llo,
                                  double Ld, RwWarp& sw) {
  FusedOut o;
  float mt = -INFINITY, tmin = INFINITY;
  int tpos = 0;
  bool nan = false;
  const float eta = (float)(ACC ? (kEx2RelErr + kCorrErr + kSum8Err) : (kEx2Raw + kSum8Err)) * 1.0001f;
  const float ka = (float)kArgRel * 1.0001f;
  // segments wholly inside an aligned row take the check-free vector loop
  const int nfull = vec ? V / RW_SEG : 0;
  // L2 prefetch LCB_RW_PF segments ahead (one bulk prefetch instruction per segment): the
  // warp's own loads then mostly hit L2, so more of the row is in flight than the registers of
  // its LDG pipeline hold (HBM still sees each byte once)
  constexpr int esz = DT == LC_BF16 ? 2 : 4;
  if (LCB_RW_PF > 0 && lane == 0 && vec)
    for (int s2 = 0; s2 < LCB_RW_PF && s2 < nfull; ++s2)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row + (size_t)s2 * RW_SEG * esz),
                   "r"((uint32_t)(RW_SEG * esz)) : "memory");
  for (int s = 0; s < nseg; ++s) {
    if (LCB_RW_PF > 0 && lane == 0 && vec && s + LCB_RW_PF < nfull)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row + (size_t)(s + LCB_RW_PF) * RW_SEG * esz),
                   "r"((uint32_t)(RW_SEG * esz)) : "memory");
    double acc = 0.0;
    float W = 0.0f, R = 0.0f;  // |a|-weighted mass (CHEAP) and rescale error, relative to mt
    // one vector of 8 ids at e0 (vmax NaN-propagating; vmin over ids < V)
    auto body = [&](const float (&vu)[8], float vmax, float vmin, int e0) {
      tmin = fminf(tmin, vmin);
      nan |= (vmax != vmax);
      if (vmax > mt) {
        if (acc > 0.0) {  // rescale the partials to the new maximum
          const float da = (mt - vmax) * Lhi;
          float f;
          if (ACC) {
            ExpCtx c2;
            c2.m = vmax;
            c2.Lhi = Lhi;
            c2.Llo = Llo;
            f = fast_exp(c2, mt);
          } else {
            f = ex2_approx(da);
          }
          const float epsf = eta + (ACC ? 0.0f : ka * -da);
          R = (R + (float)acc * epsf) * f;
          W *= f;
          acc *= (double)f;
        }
        mt = vmax;
        tpos = e0;
      }
      float ef[8], aw[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (ACC) {
          if (j & 1) continue;  // (pairs: the packed fast_exp2, bit-identical to fast_exp)
          const float2 e2 = fast_exp2(mt, Lhi, Llo, make_float2(vu[j], vu[j + 1]));
          ef[j] = e2.x;
          ef[j + 1] = e2.y;
        } else {
          const float a = (vu[j] - mt) * Lhi;
          ef[j] = ex2_approx(a);  // -inf -> +0
          aw[j] = a;
        }
      }
      // balanced 3-level fp32 tree over the 8 (kSum8Err), two lanes per packed FADD2
      const float2 s2 = f2add(f2add(make_float2(ef[0], ef[1]), make_float2(ef[2], ef[3])),
                              f2add(make_float2(ef[4], ef[5]), make_float2(ef[6], ef[7])));
      const float s8 = s2.x + s2.y;
      if (mt > -INFINITY) {  // (all -inf so far: z - mt is NaN)
        if (!ACC) {
          // CHEAP: W = sum of e*|a| (NaN once a -inf is seen: replaced at the segment end)
#pragma unroll
          for (int j = 0; j < 8; ++j) W = fmaf(ef[j], -aw[j], W);
        }
        acc += (double)s8;
      }
    };
    if (s < nfull) {
#ifndef LCB_RW_UNRF_F32
#define LCB_RW_UNRF_F32 4  // (6 spills: 10.2M rows/s)
#endif
      constexpr int UNRF = (DT == LC_BF16) ? 8 : LCB_RW_UNRF_F32;  // 128 B per lane in flight
#pragma unroll 1
      for (int st = 0; st < RW_SEGSTEPS; st += UNRF) {
        // raw vector loads first (memory-level parallelism), unpacked one vector at a time
        uint4 raw[UNRF][DT == LC_BF16 ? 1 : 2];
#pragma unroll
        for (int u = 0; u < UNRF; ++u) {
          const int e0 = s * RW_SEG + 256 * (st + u) + 8 * lane;
          if (DT == LC_BF16) {
            raw[u][0] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(row) + e0));
          } else {
            raw[u][0] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(row) + e0));
            raw[u][DT == LC_BF16 ? 0 : 1] =
                __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(row) + e0 + 4));
          }
        }
#pragma unroll
        for (int u = 0; u < UNRF; ++u) {
          const int e0 = s * RW_SEG + 256 * (st + u) + 8 * lane;
          float vv[8];
          float vmax, vmin;
          if (DT == LC_BF16) {
            // packed bf16x2 max (NaN-propagating) / min over the 8 values
            const uint32_t w[4] = {raw[u][0].x, raw[u][0].y, raw[u][0].z, raw[u][0].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              vv[2 * j] = __uint_as_float(w[j] << 16);
              vv[2 * j + 1] = __uint_as_float(w[j] & 0xffff0000u);
            }
            uint32_t x01, x23, x, n01, n23, n;
            asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(x01) : "r"(w[0]), "r"(w[1]));
            asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(x23) : "r"(w[2]), "r"(w[3]));
            asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(x) : "r"(x01), "r"(x23));
            asm("min.bf16x2 %0, %1, %2;" : "=r"(n01) : "r"(w[0]), "r"(w[1]));
            asm("min.bf16x2 %0, %1, %2;" : "=r"(n23) : "r"(w[2]), "r"(w[3]));
            asm("min.bf16x2 %0, %1, %2;" : "=r"(n) : "r"(n01), "r"(n23));
            vmax = max_nan(__uint_as_float(x << 16), __uint_as_float(x & 0xffff0000u));
            vmin = fminf(__uint_as_float(n << 16), __uint_as_float(n & 0xffff0000u));
          } else {
            const uint4 a = raw[u][0], b = raw[u][DT == LC_BF16 ? 0 : 1];
            vv[0] = __uint_as_float(a.x); vv[1] = __uint_as_float(a.y);
            vv[2] = __uint_as_float(a.z); vv[3] = __uint_as_float(a.w);
            vv[4] = __uint_as_float(b.x); vv[5] = __uint_as_float(b.y);
            vv[6] = __uint_as_float(b.z); vv[7] = __uint_as_float(b.w);
            vmax = max_nan(max_nan(max_nan(vv[0], vv[1]), max_nan(vv[2], vv[3])),
                           max_nan(max_nan(vv[4], vv[5]), max_nan(vv[6], vv[7])));
            vmin = fminf(fminf(fminf(vv[0], vv[1]), fminf(vv[2], vv[3])),
                         fminf(fminf(vv[4], vv[5]), fminf(vv[6], vv[7])));
          }
          body(vv, vmax, vmin, e0);
        }
      }
    } else {
      // tail segment / unaligned row: one generic vector at a time
#pragma unroll 1
      for (int st = 0; st < RW_SEGSTEPS && s * RW_SEG + 256 * st < V; ++st) {
        const int e0 = s * RW_SEG + 256 * st + 8 * lane;
        if (e0 >= V) continue;  // past the row (its -inf padding would make W NaN)
        float vv[8];
        load8<DT>(row, e0, V, vec, vv);
        float vmax = vv[0], vmin = INFINITY;
#pragma unroll
        for (int j = 1; j < 8; ++j) vmax = max_nan(vmax, vv[j]);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (e0 + j < V) vmin = fminf(vmin, vv[j]);
        body(vv, vmax, vmin, e0);
      }
    }
    // segment end: combine at the warp's running maximum.  A -inf element made W NaN:
    // bound it by 150 octaves per unit of mass instead (beyond that e < 2^-150: absolute,
    // in absE)
    if (!ACC && W != W) W = 150.0f * (float)acc * 1.001f;
    const float ms = warp_max(mt);
    float g = 1.0f, epsg = 0.0f;
    if (mt < ms && acc > 0.0) {
      const float da = (mt - ms) * Lhi;
      if (ACC) {
        ExpCtx c2;
        c2.m = ms;
        c2.Lhi = Lhi;
        c2.Llo = Llo;
        g = fast_exp(c2, mt);
      } else {
        g = ex2_approx(da);
      }
      epsg = eta + (ACC ? 0.0f : ka * -da);
    }
    const double sa = warp_sum(acc * (double)g);
    const double sE = warp_sum((double)g * (acc * (double)(eta + epsg) + (double)R + (double)(ka * W)));
    if (lane == 0) {
      sw.seg[s] = sa;
      sw.segE[s] = sE;
      sw.segm[s] = ms;
    }
  }
  __syncwarp();
  o.tmax = mt;
  o.tmin = tmin;
  o.tpos = tpos;
  o.nan = __any_sync(0xffffffffu, nan);
  // rescale the segments to the row maximum (fp64 exp2: relative error ~2^-51)
  const float m = warp_max(mt);
  double S = 0.0, ES = 0.0, rel = 0.0;
  if (lane < nseg) {
    const double h = exp2(((double)sw.segm[lane] - (double)m) * Ld);
    const double x = sw.seg[lane] * h;
    const double e = sw.segE[lane] * h + x * 1e-15;
    sw.seg[lane] = x;
    S = x;
    ES = e;
    rel = x > 0.0 ? e / x : 0.0;
  }
  __syncwarp();
  o.S = warp_sum(S);
  o.ES = warp_sum(ES);
  o.relmax = rel;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) o.relmax = fmax(o.relmax, __shfl_xor_sync(0xffffffffu, o.relmax, off));
  return o;
}

// e-function variants: 0 CHEAP (truncated rows), 1 ACCURATE (untruncated), 2 PRECISE (lite)
template <int EM>
__device__ __forceinline__ double rw_e(const ExpCtx& ec, float z, const double* t16, float& aw) {
  if (EM == 2) {
    aw = 0.0f;
    return lite_exp(ec, z, t16);
  } else if (EM == 1) {
    aw = 0.0f;
    return (double)fast_exp(ec, z);
  } else {
    float a;
    const float e = cheap_exp(ec, z, a);
    aw = -a * e;
    return (double)e;
  }
}

// One pass over the row; seg[s] = sum of e over the segment's ids; returns the
// |a|-weighted W (CHEAP only).  FAST variants sum 8 values in fp32 pairs then in
// fp64 (matched by the rescan).
template <int DT, int EM>
__device__ double rw_seg_pass(const char* row, int V, int nseg, bool vec, int lane, const ExpCtx& ec,
                              const double* t16, double* seg) {
  __syncwarp();  // earlier reads of seg (a previous tier's draws) before this pass rewrites it
  float Wl = 0.0f;
  for (int s = 0; s < nseg; ++s) {
    double acc = 0.0;
    const int s0 = s * RW_SEG;
#pragma unroll 4
    for (int st = 0; st < RW_SEGSTEPS; ++st) {
      const int e0 = s0 + 256 * st + 8 * lane;
      float v[8];
      load8<DT>(row, e0, V, vec, v);
      double e8 = 0.0;
      float ef[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float aw;
        const double e = rw_e<EM>(ec, v[j], t16, aw);
        if (EM == 2) e8 += e;
        else ef[j] = (float)e;
        Wl += aw;
      }
      if (EM != 2) e8 = (double)(((ef[0] + ef[1]) + (ef[2] + ef[3])) + ((ef[4] + ef[5]) + (ef[6] + ef[7])));
      acc += e8;
    }
    acc = warp_sum(acc);
    if (lane == 0) seg[s] = acc;
  }
  __syncwarp();
  return warp_sum((double)Wl) * 1.001;
}

// Big-nucleus histogram: bin b (1/32 octave below the max) accumulates
// q = e * 2^(b/32) = ex2(a + b/32) in per-bin relative fixed point (the sum
// a + b/32 is exact: a and -b/32 are within a factor 2).  Out of line: its own
// register budget.
// 8 consecutive logits at an aligned, in-range e0 (no checks)
template <int DT>
__device__ __forceinline__ void load8_full(const char* row, int e0, float v[8]) {
  if (DT == LC_BF16) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(row) + e0));
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[2 * j] = __uint_as_float(w[j] << 16);
      v[2 * j + 1] = __uint_as_float(w[j] & 0xffff0000u);
    }
  } else {
    const float4 a = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(row) + e0));
    const float4 b = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(row) + e0 + 4));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}

template <int DT>
__device__ __noinline__ void rw_hist_pass(const char* row, int V, bool vec, int lane, float m, float Lhi, float qscale,
                                          uint32_t hist_s) {
  auto add = [&](float z) {
    const float a = fmaxf((z - m) * Lhi, -200.0f);
    const int b = rw_bin(a);
    const uint32_t q = __float2uint_rn(ex2_approx(fmaf((float)b, 1.0f / RW_BPO, a)) * qscale);
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(hist_s + 4u * (uint32_t)b), "r"(q) : "memory");
  };
  const int vfull = vec ? (V / 1024) * 1024 : 0;
  for (int base = 0; base < vfull; base += 1024) {  // four vectors per lane in flight, no checks
    float v[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u) load8_full<DT>(row, base + 256 * u + 8 * lane, v[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) add(v[u][j]);
  }
#pragma unroll 1
  for (int base = vfull; base < V; base += 256) {  // tail: ids >= V read as -inf (q = 0)
    float v[8];
    load8<DT>(row, base + 8 * lane, V, vec, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) add(v[j]);
  }
}

// Big-nucleus kept list: ids with z >= zhi (bin <= bhi) in id order, bracket
// members (z < zab) flagged in bit 31 and their keys appended to sw.cand.
// Returns the list length (entries beyond cap are not written).
template <int DT>
__device__ __noinline__ int rw_list_pass(const char* row, int V, bool vec, int lane, float zhi, float zab, int2* L_iz,
                                         int cap, RwWarp& sw, int& ovf) {
  int wn = 0;
  // NV vectors (256 ids each) per step; ids >= V read as -inf (never >= zhi)
  auto step = [&](const float (&v)[2][8], int nv, int base) {
    unsigned lm[2] = {0u, 0u}, bm[2] = {0u, 0u};
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        lm[u] |= (v[u][j] >= zhi ? 1u : 0u) << j;
        bm[u] |= (v[u][j] >= zhi && v[u][j] < zab ? 1u : 0u) << j;
      }
    if (nv < 2) lm[1] = bm[1] = 0u;
    // both vectors' counts in one scan (16-bit halves)
    const int c = __popc(lm[0]) | (__popc(lm[1]) << 16);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    const int t0 = tot & 0xffff;
    const int pos0[2] = {wn + (incl & 0xffff) - (c & 0xffff), wn + t0 + (incl >> 16) - (c >> 16)};
    const int e0[2] = {base + 8 * lane, base + 256 + 8 * lane};
    if (wn + t0 + (tot >> 16) <= cap) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        int pos = pos0[u];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if ((lm[u] >> j) & 1u) {
            L_iz[pos] = make_int2(e0[u] + j + (int)(((bm[u] >> j) & 1u) << 31), __float_as_int(v[u][j]));
            ++pos;
          }
      }
    }
    // bracket keys use the LIST POSITION instead of the id: the list is id-ordered,
    // so (z desc, position asc) is the reference's (p desc, id asc) order
    if (bm[0] | bm[1]) {
      int p2 = atomicAdd(&sw.isc[0], __popc(bm[0]) + __popc(bm[1]));
#pragma unroll
      for (int u = 0; u < 2; ++u)
        for (unsigned b = bm[u]; b; b &= b - 1u) {
          const int j = __ffs(b) - 1;
          if (p2 < RW_CAND) sw.cand[p2] = cand_key(v[u][j], pos0[u] + __popc(lm[u] & ((1u << j) - 1u)));
          else ovf = 1;
          ++p2;
        }
    }
    wn += t0 + (tot >> 16);
  };
  const int vfull = vec ? (V / 512) * 512 : 0;
  for (int base = 0; base < vfull && wn <= cap; base += 512) {  // two vectors per lane, no checks
    float v[2][8];
    load8_full<DT>(row, base + 8 * lane, v[0]);
    load8_full<DT>(row, base + 256 + 8 * lane, v[1]);
    step(v, 2, base);
  }
#pragma unroll 1
  for (int base = vfull; base < V && wn <= cap; base += 256) {  // tail, one vector per step
    float v[2][8];
    load8<DT>(row, base + 8 * lane, V, vec, v[0]);
    step(v, 1, base);
  }
  return wn;
}

#ifdef LCB_RW_DEBUG
// debug build only (LCB_NVCC_EXTRA=-DLCB_RW_DEBUG): per-task trace of the row-warp kernel
__device__ double g_rw_dbg[256][12];
#define RW_DBG(k, x) \
  do {                                                          \
    if (lane == 0 && task_id < 256) g_rw_dbg[task_id][k] = (double)(x); \
  } while (0)
#else
#define RW_DBG(k, x) \
  do {              \
  } while (0)
#endif

struct RwScratch {
  int2* iz;    // [warps][cap] kept list in id order: {id | bracket-member bit 31, z bits}
  double* e;   // [warps][cap] fp64-lite e
  int cap;
  int* next;   // dynamic task counter
  int* q_cta;  // [0] = count, [1..] task ids with an effective top-k (CTA kernel)
};

template <int DT, int MINB>
__global__ void __launch_bounds__(RW_THREADS, MINB)
rowwarp_kernel(const char* __restrict__ rows, int64_t row_bytes, int Vdef, const lc_task* __restrict__ tasks,
               int n_tasks, CacheMap cm, DrawIO io, int* q_exact, unsigned long long* counters, RwScratch scr,
               int force) {
  extern __shared__ __align__(16) unsigned char rw_smraw[];
  RwSmem& smem = *reinterpret_cast<RwSmem*>(rw_smraw);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  RwWarp& sw = smem.w[wid];
  if (threadIdx.x < 16) smem.t16[threadIdx.x] = exp2((double)threadIdx.x / 16.0);
  if (lane == 0) sw.isc[0] = 0;
  __syncthreads();
  const int gw = blockIdx.x * RW_WARPS + wid;
  int2* L_iz = scr.iz + (int64_t)gw * scr.cap;
  double* L_e = scr.e + (int64_t)gw * scr.cap;

  for (;;) {
    // (the previous task's reads of the warp's shared scratch are ordered before this task's
    // writes: lanes may otherwise run ahead under independent thread scheduling)
    __syncwarp();
    // dynamic scheduling: tasks differ wildly in cost (fast exit vs big nucleus)
    int task_id = 0;
    if (lane == 0) task_id = atomicAdd(scr.next, 1);
    task_id = __shfl_sync(0xffffffffu, task_id, 0);
    if (task_id >= n_tasks) break;
    const lc_task tk = tasks[task_id];
    if (tk.draw_end <= tk.draw_begin) continue;
    const int Vt = tk.vocab > 0 ? tk.vocab : Vdef;
    if (tk.top_k > 0 && tk.top_k < Vt) {  // top-k: queued for the CTA kernel
      if (lane == 0) {
        const int pos = atomicAdd(scr.q_cta, 1);
        scr.q_cta[1 + pos] = task_id;
      }
      continue;
    }
    TaskView tv;
    if (!resolve_task(tk, rows, row_bytes, Vdef, cm, tv)) {
      for (int64_t d = tv.d0 + lane; d < tv.d1; d += 32) {
        io.token[d] = -1;
        if (io.flags) io.flags[d] = LC_DRAW_BAD_ROW;
      }
      if (lane == 0) {
        atomicAdd(&counters[2], 1ull);
        set_kept(io, task_id, -1);
      }
      continue;
    }
    if (force == 2) {  // test hook: everything to the EXACT tier
      if (lane == 0) {
        const int pos = atomicAdd(q_exact, 1);
        q_exact[1 + pos] = task_id;
      }
      continue;
    }
    const int V = tv.V;
    const bool vec = ((reinterpret_cast<uintptr_t>(tv.row) & 15) == 0);
    const int nseg = (V + RW_SEG - 1) / RW_SEG;
    auto write_all_w = [&](int tok, uint8_t flag) {
      for (int64_t d = tv.d0 + lane; d < tv.d1; d += 32) {
        io.token[d] = tok;
        if (io.flags) io.flags[d] = flag;
      }
    };

    // ---------------- one read of the row: max / min / NaN (+ mass for T > 0)
    float tmax = -INFINITY, tmin = INFINITY;
    int tpos = 0;
    FusedOut fo{};
    double Ld = 0.0;
    float Lhi = 0.0f, Llo = 0.0f;
    if (tv.T == 0.0) {
      phase_a_pos<DT>(tv.row, V, vec, lane, tmax, tmin, tpos);
    } else {
      Ld = tv.Ld;  // log2(e) / T, divided once per task when it was resolved
      Lhi = (float)Ld;
      Llo = (float)(Ld - (double)Lhi);
      fo = tv.trunc ? rw_fused_pass<DT, false>(tv.row, V, nseg, vec, lane, Lhi, Llo, Ld, sw)
                    : rw_fused_pass<DT, true>(tv.row, V, nseg, vec, lane, Lhi, Llo, Ld, sw);
      tmax = fo.nan ? NAN : fo.tmax;
      tmin = fo.tmin;
      tpos = fo.tpos;
    }
    const bool bad = __any_sync(0xffffffffu, (tmax != tmax) || (tmin != tmin));
    if (bad) tmax = -INFINITY;
    const float m = warp_max(tmax);
    const float zmin = -warp_max(-tmin);
    if (bad || !(m > -INFINITY) || !(m < INFINITY)) {
      write_all_w(-1, LC_DRAW_BAD_ROW);
      if (lane == 0) {
        atomicAdd(&counters[2], 1ull);
        set_kept(io, task_id, -1);
      }
      continue;
    }
    // first argmax: lanes holding m reload the first vector that held their maximum
    auto first_argmax = [&]() -> int {
      int best = INT_MAX;
      if (tmax == m) {
        float v[8];
        load8<DT>(tv.row, tpos, V, vec, v);
#pragma unroll
        for (int j = 7; j >= 0; --j)
          if (v[j] == m) best = tpos + j;
      }
      return warp_min_int(best);
    };
    if (tv.T == 0.0) {
      const int a = first_argmax();
      write_all_w(a, 0);
      if (lane == 0) set_kept(io, task_id, greedy_kept(V, tv.topk, tv.topp));
      continue;
    }
    ExpCtx ec;
    ec.m = m;
    ec.T = tv.T;
    ec.mT = __ddiv_rn((double)m, tv.T);
    ec.md = (double)m;
    ec.Lhi = Lhi;
    ec.Llo = Llo;
    ec.L16 = 16.0 * Ld;
    const double zabs = fmax(fabs((double)m), isfinite(zmin) ? fabs((double)zmin) : fabs((double)m));
    const double zT = zabs / tv.T;
    const bool sane = ec.Lhi < 1e20f && ec.Lhi > 1e-20f && fabsf(m) * ec.Lhi < 1e30f && zT < 1e15;
    const double relArg = 4.440892098500626e-16 * 2.0 * zT;
    const double relRef = (double)(2 * V + 64) * kEps64;
    const bool accurate = !tv.trunc;  // untruncated: the draw itself needs tight per-element errors
    // relative bound of the fp64-lite e's (kept lists, PRECISE pass) vs the reference's e's
    const double relLite = kLiteErr + 2.0 * kRefExpErr + relArg + (double)(V + 16) * kEps64;

    // ---------------- phase B: segment masses (+ |a|-weighted bound for the cheap exp)
    bool done = false, to_exact = !sane;
    int big_state = 0;  // 0 not built, 1 built, -1 failed
    int blo = 0, bhi = 0, nb = 0, nl = 0;
    double Mab = 0.0;  // fp64-lite mass of the list entries above the bracket

    for (int pass = force == 1 ? 1 : 0; pass < 2 && !done && !to_exact; ++pass) {
      const bool precise = pass == 1;
      const uint8_t tier_flag = precise ? LC_DRAW_PRECISE : 0;
      if (precise) {
        if (lane == 0) atomicAdd(&counters[0], 1ull);
        rw_seg_pass<DT, 2>(tv.row, V, nseg, vec, lane, ec, smem.t16, sw.seg);
      }
      double S = 0.0;
      for (int s = 0; s < nseg; ++s) S += sw.seg[s];
      RW_DBG(0, S);
      RW_DBG(1, fo.ES);
      RW_DBG(2, fo.relmax);
      RW_DBG(3, ec.m);
      RW_DBG(4, zmin);
      // FAST: the fused pass's bound (element exps, rescales, pair sums) + the reference's
      // argument/exp rounding + fp64 accumulation; PRECISE: lite_exp's
      const double relCommon = kRefExpErr + relArg + (double)(V + 16) * kEps64;
      const double relE = precise ? relLite : fo.relmax + relCommon;
      const double absE = precise ? (double)V * 1e-300 : (double)V * 2.4e-38;
      const double E_S = precise ? S * relE + absE : fo.ES + S * relCommon + absE;

      bool big = false;
      unsigned long long kcut = 0ull;
      int cut = -1;
      if (tv.trunc && tv.topp < 1.0) {
        const double pmax_lo = (1.0 / (S + E_S)) * (1.0 - relRef);
        if (pmax_lo > tv.topp) {  // nucleus = {first argmax}
          write_all_w(first_argmax(), tier_flag);
          if (lane == 0) set_kept(io, task_id, 1);
          done = true;
          break;
        }
        const double P = tv.topp * S;
        if (big_state == 0) {
          // histogram: per-bin relative fixed point (bin b holds e in (2^-(b+1)/32, 2^-b/32]);
          // q = e * 2^(b/32) = ex2(a + b/32), the sum exact (a and -b/32 within a factor 2)
          for (int i = lane; i < RW_NB; i += 32) sw.hist[i] = 0u;
          __syncwarp();
          const int lgV = 32 - __clz(V + 1);
          const float qscale = ldexpf(1.0f, 31 - lgV);
          rw_hist_pass<DT>(tv.row, V, vec, lane, ec.m, ec.Lhi, qscale, (uint32_t)__cvta_generic_to_shared(sw.hist));
          __syncwarp();
          // bracket of bins that can hold the cut
          const double inv = 1.0 / (double)qscale;
          const double qrel = ldexp(1.0, lgV - 31) * 1.2 + kEx2Raw + kArgRel * 33.0 + 1e-7;
          const double qerr = qrel * S + 2.0 * E_S + P * relRef;
          double cum = 0.0;
          blo = RW_NB - 1;
          bhi = RW_NB - 1;
          bool got_lo = false;
          for (int b0 = 0; b0 < RW_NB; b0 += 32) {
            const double hb = (double)sw.hist[b0 + lane] * inv * exp2(-(double)(b0 + lane) / (double)RW_BPO);
            const double incl = cum + warp_incl_scan(hb);
            const unsigned lo_m = __ballot_sync(0xffffffffu, incl >= P - qerr);
            const unsigned hi_m = __ballot_sync(0xffffffffu, incl >= P + qerr);
            if (!got_lo && lo_m) {
              blo = b0 + __ffs(lo_m) - 1;
              got_lo = true;
            }
            if (hi_m) {
              bhi = b0 + __ffs(hi_m) - 1;
              break;
            }
            cum = __shfl_sync(0xffffffffu, incl, 31);
          }
          big_state = (bhi >= RW_NB - 1) ? -1 : 1;  // a cut in the catch-all bin -> EXACT
          RW_DBG(5, blo);
          RW_DBG(6, bhi);
          if (big_state > 0) {
            // kept list: ids with bin <= bhi in id order (bracket members flagged); bracket
            // keys also go to the smem candidate list for the exact sort.  Bins are
            // monotone in z: bin <= bhi <=> z >= zhi, bin < blo <=> z >= zab.
            const float zhi = rw_zthr(ec, bhi), zab = rw_zthr(ec, blo - 1);
            __syncwarp();
            int ovf = 0;
            const int wn = rw_list_pass<DT>(tv.row, V, vec, lane, zhi, zab, L_iz, scr.cap, sw, ovf);
            __syncwarp();
            nb = sw.isc[0];
            nl = wn;
            RW_DBG(7, nb);
            RW_DBG(8, nl);
            RW_DBG(9, ovf);
            if (__any_sync(0xffffffffu, ovf) || nb > RW_CAND || nl > scr.cap) {
              big_state = -1;
            } else {
              // fp64-lite e of the list (dense, one 32-entry chunk per step); per-chunk mass
              // above the bracket (bracket members are added after the cut) and its total
              double acc = 0.0;
              const int nch = (nl + 31) / 32;
              if (nch > RW_NCH) big_state = -1;
              for (int c = 0; c < nch && big_state > 0; c += 2) {  // two chunks in flight
                const int i0 = c * 32 + lane, i1 = i0 + 32;
                const int2 iz0 = i0 < nl ? L_iz[i0] : make_int2(0, __float_as_int(-INFINITY));
                const int2 iz1 = i1 < nl ? L_iz[i1] : make_int2(0, __float_as_int(-INFINITY));
                const double e0 = lite_exp(ec, __int_as_float(iz0.y), smem.t16);
                const double e1 = lite_exp(ec, __int_as_float(iz1.y), smem.t16);
                if (i0 < nl) L_e[i0] = e0;
                if (i1 < nl) L_e[i1] = e1;
                const double ea0 = iz0.x >= 0 ? e0 : 0.0, ea1 = iz1.x >= 0 ? e1 : 0.0;
                double cs0 = ea0, cs1 = ea1;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                  cs0 += __shfl_xor_sync(0xffffffffu, cs0, o);
                  cs1 += __shfl_xor_sync(0xffffffffu, cs1, o);
                }
                if (lane == 0) {
                  sw.chunk_above[c] = cs0;
                  if (c + 1 < nch) sw.chunk_above[c + 1] = cs1;
                }
                acc += ea0 + ea1;
              }
              Mab = warp_sum(acc);
              // rank sort of the bracket keys (z desc, id asc) through ce[] as scratch
              unsigned long long* tmpk = reinterpret_cast<unsigned long long*>(sw.ce);
              for (int i = lane; i < nb; i += 32) {
                const unsigned long long kk = sw.cand[i];
                int rank = 0;
                for (int j = 0; j < nb; ++j) rank += (sw.cand[j] > kk);
                tmpk[rank] = kk;
              }
              __syncwarp();
              for (int i = lane; i < nb; i += 32) sw.cand[i] = tmpk[i];
              __syncwarp();
              for (int i = lane; i < nb; i += 32) sw.ce[i] = ref_exp(ec, cand_z(sw.cand[i]));
            }
          }
          __syncwarp();
          if (lane == 0) sw.isc[0] = 0;
          __syncwarp();
        }
        if (big_state < 0) {
          to_exact = true;
          if (lane == 0) atomicAdd(&counters[7], 1ull);
          break;
        }
        // cut inside the bracket: csum (precise e's) from the mass above it
        const double EMab = Mab * relLite;
        cut = -1;
        bool unc = Mab >= P - tv.topp * E_S - EMab;  // the cut would lie above the bracket
        double off = Mab;
        for (int i0 = 0; i0 < nb && !unc; i0 += 32) {
          const int i = i0 + lane;
          const double e = i < nb ? sw.ce[i] : 0.0;
          const double c = off + warp_incl_scan(e), prev = c - e;
          const double tol = tv.topp * E_S + EMab + c * relRef;
          const unsigned hm = __ballot_sync(0xffffffffu, i < nb && c >= P - tol);
          if (hm) {
            const int hl = __ffs(hm) - 1;
            cut = i0 + hl;
            const bool ok = (c - P > tol && P - prev > tol);
            unc = !__shfl_sync(0xffffffffu, ok, hl);
            break;
          }
          off = __shfl_sync(0xffffffffu, c, 31);
        }
        if (cut < 0) unc = true;
        if (!unc) {
          bool bad_order = false;
          for (int i = max(cut, 1) + lane; i <= min(cut + 1, nb - 1); i += 32) {
            const float za = cand_z(sw.cand[i - 1]), zb = cand_z(sw.cand[i]);
            if (za != zb) {
              const double da = __ddiv_rn((double)za, tv.T), db = __ddiv_rn((double)zb, tv.T);
              if (da - db <= fmax(fabs(da), fabs(ec.mT)) * 8.0 * kEps64) bad_order = true;
            }
          }
          unc = __any_sync(0xffffffffu, bad_order);
        }
        if (unc) {
          if (lane == 0 && !precise) atomicAdd(&counters[4], 1ull);
          continue;
        }
        big = true;
        kcut = sw.cand[cut];
      }

      int need = 0;
      if (big) {
        // ---------------- draws over the kept list (precise e's, id order)
        // chunk sums = mass above the bracket + the kept bracket members (located by binary
        // search on the id-ordered list); each lane then locates one target on its own
        double* csum = sw.chunk_tot;
        const int nch = (nl + 31) / 32;
        {
          for (int c = lane; c < nch; c += 32) csum[c] = sw.chunk_above[c];
          __syncwarp();
          for (int b = lane; b <= cut; b += 32) {
            const int pos = cand_id(sw.cand[b]);  // list position (see the list pass)
            atomicAdd(&csum[pos / 32], L_e[pos]);
          }
          __syncwarp();
          if (lane == 0) {  // exclusive prefix over chunks (sequential: exact order)
            double c = 0.0;
            for (int q = 0; q < nch; ++q) {
              const double x = csum[q];
              csum[q] = c;
              c += x;
            }
            csum[nch] = c;
          }
          __syncwarp();
          const double K = csum[nch];
          const double relD = relLite + (double)(nl + 64) * 4.0 * kEps64;
          for (int64_t d = tv.d0 + lane; d < tv.d1; d += 32) {
            const double u = draw_u(io, d, tv);
            const double tk = u * K;
            int found = -1;
            double flo = 0.0, fhi = 0.0;
            if (tk < K) {
              int lo = 0, hi = nch;  // last chunk with prefix <= tk
              while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (csum[mid] <= tk) lo = mid;
                else hi = mid;
              }
              double c = csum[lo];
              const int i0 = lo * 32, i1 = min(nl, i0 + 32);
              for (int i = i0; i < i1; ++i) {
                const int2 iz = L_iz[i];
                const int idf = iz.x;
                double e = L_e[i];
                if (idf < 0 && cand_key(__int_as_float(iz.y), i) < kcut) e = 0.0;  // beyond the cut
                const double nc = c + e;
                if (e > 0.0 && tk < nc) {
                  found = idf & 0x7fffffff;
                  flo = c;
                  fhi = nc;
                  break;
                }
                c = nc;
              }
            }
            const double tlo = relD * ((1.0 - u) * flo + u * (K - flo)) + tk * relRef * 4.0;
            const double thi = relD * ((1.0 - u) * fhi + u * (K - fhi)) + tk * relRef * 4.0;
            // nothing kept precedes flo == 0: the lower boundary is exact
            const bool ok = found >= 0 && (tk - flo > tlo || flo == 0.0) && (fhi - tk > thi);
            io.token[d] = found;
            if (io.flags) io.flags[d] = tier_flag;
            need |= !ok;
          }
        }
      } else {
        // ---------------- draws over all ids: segment prefix, one rescan per segment
        if (lane == 0) {
          double c = 0.0;
          for (int s = 0; s < nseg; ++s) {
            const double x = sw.seg[s];
            sw.seg[s] = c;
            c += x;
          }
          sw.seg[nseg] = c;
        }
        __syncwarp();
        const double K = sw.seg[nseg];
        const double absD = fmax(absE, E_S - relE * S);  // absolute part of the bound (flushed mass)
        // FAST: walk e's vs fused-pass e's inside a segment (PRECISE: the same lite_exp values)
        const double relX = precise ? 0.0 : (fo.relmax + kEx2RelErr + kCorrErr + kSum8Err + relArg) * 1.01;
        for (int64_t dbase = tv.d0; dbase < tv.d1; dbase += 32) {
          const int64_t d = dbase + lane;
          double t = INFINITY, u = 0.0;
          if (d < tv.d1) {
            u = draw_u(io, d, tv);
            t = u * K;
            if (!(t < K)) need = 1;  // clamp region -> EXACT
          }
          double st = (d < tv.d1 && t < K) ? t : INFINITY;
          int ssrc = lane;
#pragma unroll
          for (int k2 = 2; k2 <= 32; k2 <<= 1) {
#pragma unroll
            for (int j2 = k2 >> 1; j2 > 0; j2 >>= 1) {
              const double ot = __shfl_xor_sync(0xffffffffu, st, j2);
              const int os = __shfl_xor_sync(0xffffffffu, ssrc, j2);
              const bool asc = (lane & k2) == 0 || k2 == 32;
              const bool lower = (lane & j2) == 0;
              const bool take =
                  (lower == asc) ? (ot < st || (ot == st && os < ssrc)) : (ot > st || (ot == st && os > ssrc));
              if (take) {
                st = ot;
                ssrc = os;
              }
            }
          }
          const double su = __shfl_sync(0xffffffffu, u, ssrc);
          const int ntar = __popc(__ballot_sync(0xffffffffu, st < INFINITY));
          int k = 0;
          while (k < ntar) {
            const double tk0 = __shfl_sync(0xffffffffu, st, k);
            int s = 0;
            while (s + 1 < nseg && sw.seg[s + 1] <= tk0) ++s;
            double off = sw.seg[s];
            const double seg0 = off;  // the segment's prefix (from the fused pass)
            const double send = sw.seg[s + 1];
            for (int stp = 0; stp < RW_SEGSTEPS && k < ntar; ++stp) {
              const int my0 = s * RW_SEG + 256 * stp + 8 * lane;
              float v[8];
              load8<DT>(tv.row, my0, V, vec, v);
              double ev[8];
              double ls;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                float aw;
                ev[j] = precise ? rw_e<2>(ec, v[j], smem.t16, aw)
                                : (accurate ? rw_e<1>(ec, v[j], smem.t16, aw) : rw_e<0>(ec, v[j], smem.t16, aw));
              }
              if (!precise) {  // the FAST segment sums used the fp32 pair-sum association
                float f[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) f[j] = (float)ev[j];
                const float2 s2 = f2add(f2add(make_float2(f[0], f[1]), make_float2(f[2], f[3])),
                                        f2add(make_float2(f[4], f[5]), make_float2(f[6], f[7])));
                ls = (double)(s2.x + s2.y);  // (the fused pass's association)
              } else {
                ls = 0.0;
#pragma unroll
                for (int j = 0; j < 8; ++j) ls += ev[j];
              }
              const double x = warp_incl_scan(ls);
              const double tot = __shfl_sync(0xffffffffu, x, 31);
              while (k < ntar) {
                const double tk = __shfl_sync(0xffffffffu, st, k);
                if (!(tk < off + tot) && !(stp == RW_SEGSTEPS - 1 && tk < send)) break;
                const unsigned hm = __ballot_sync(0xffffffffu, (ls > 0.0) && (tk < off + x));
                int found = -1;
                double flo = 0.0, fhi = 0.0, gm = 0.0;
                if (hm) {
                  const int hl = __ffs(hm) - 1;
                  if (lane == hl) {
                    double c = off + (x - ls);
                    for (int j = 0; j < 8; ++j) {
                      const double nc = c + ev[j];
                      if (ev[j] > 0.0 && tk < nc) {
                        found = my0 + j;
                        flo = c;
                        fhi = nc;
                        break;
                      }
                      c = nc;
                    }
                  }
                  found = __shfl_sync(0xffffffffu, found, hl);
                  flo = __shfl_sync(0xffffffffu, flo, hl);
                  fhi = __shfl_sync(0xffffffffu, fhi, hl);
                  gm = precise ? 0.0 : __shfl_sync(0xffffffffu, ls, hl);  // (fp32-tree group sum)
                }
                const double uu = __shfl_sync(0xffffffffu, su, k);
                const int src = __shfl_sync(0xffffffffu, ssrc, k);
                if (lane == 0) {
                  // correlated bound over the segment prefixes (the fused pass's e's on both sides),
                  // plus the uncorrelated part: inside segment s the walk sums its own e's (relative
                  // to the row max), not the fused pass's (relative to running maxima, rescaled), so
                  // their difference is bounded by both errors times the walked mass
                  const double tlo = relE * ((1.0 - uu) * flo + uu * (K - flo)) + relX * (flo - seg0) + absD +
                                     tk * relRef * 4.0 + kSum8Err * gm;
                  const double thi = relE * ((1.0 - uu) * fhi + uu * (K - fhi)) + relX * (fhi - seg0) + absD +
                                     tk * relRef * 4.0 + kSum8Err * gm;
                  const bool ok = found >= 0 && (tk - flo > tlo || (precise && flo == 0.0)) && (fhi - tk > thi);
                  io.token[dbase + src] = found;
                  if (io.flags) io.flags[dbase + src] = tier_flag;
                  need |= !ok;
                }
                ++k;
              }
              off += tot;
            }
            while (k < ntar && __shfl_sync(0xffffffffu, st, k) < send) {
              const int src = __shfl_sync(0xffffffffu, ssrc, k);
              if (lane == 0) {
                io.token[dbase + src] = -1;
                need = 1;
              }
              ++k;
            }
          }
        }
      }
      need = __any_sync(0xffffffffu, need);
      if (!need) {
        done = true;
        // big nucleus: the list entries above the bracket + bracket members 0..cut (sorted);
        // otherwise untruncated (identity)
        if (lane == 0) set_kept(io, task_id, big ? (nl - nb) + cut + 1 : V);
      } else if (lane == 0 && !precise) {
        atomicAdd(&counters[5], 1ull);
      }
    }
    if (!done && lane == 0) {
      const int pos = atomicAdd(q_exact, 1);
      q_exact[1 + pos] = task_id;
      atomicAdd(&counters[3], 1ull);
    }
  }
}

// ============================== EXACT kernel ==============================
// numpy emulation (pairwise_seq in lc_numpy.cuh).

constexpr int EX_THREADS = 256;
constexpr int EX_CAND = 8192;  // exact-tier candidate set in shared memory (96 KB, dynamic)

template <int DT>
__global__ void __launch_bounds__(EX_THREADS)
exact_kernel(const char* __restrict__ rows, int64_t row_bytes, int Vdef, const lc_task* __restrict__ tasks,
             const int* __restrict__ task_list, CacheMap cm, DrawIO io, double* scratch, int32_t* iscratch,
             int64_t scr_stride, unsigned long long* counters) {
  const int ntask = task_list[0];
  double* p = scratch + (int64_t)blockIdx.x * scr_stride * 3;  // probabilities
  double* q = p + scr_stride;                                   // truncated, renormalised
  double* tmp = q + scr_stride;                                 // kept values in sorted order
  int32_t* ord = iscratch + (int64_t)blockIdx.x * scr_stride;   // kept ids in sorted order
  __shared__ float s_m;
  __shared__ double s_S;
  __shared__ int s_L;
  __shared__ double s_bp[EX_THREADS];
  __shared__ int s_bi[EX_THREADS];
  __shared__ int s_stop;
  extern __shared__ __align__(16) unsigned char ex_dyn[];
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(ex_dyn);
  int* s_id = reinterpret_cast<int*>(ex_dyn + EX_CAND * 8);
  // pairwise leaves alias the candidate arrays (never live at the same time)
  constexpr int kLeafCap = EX_CAND / 2;
  int2* s_lv = reinterpret_cast<int2*>(ex_dyn);
  double* s_ls = reinterpret_cast<double*>(ex_dyn + kLeafCap * 8);
  __shared__ double s_bc;
  __shared__ int s_nl;
  const int tid = threadIdx.x;
  for (int ti = blockIdx.x; ti < ntask; ti += gridDim.x) {
    const int task_id = task_list[1 + ti];
    TaskView tv;
    if (tasks[task_id].draw_end <= tasks[task_id].draw_begin) continue;
    if (!resolve_task(tasks[task_id], rows, row_bytes, Vdef, cm, tv)) continue;
    const int V = tv.V;
    // max (fp32 exact)
    float mloc = -INFINITY;
    for (int i = tid; i < V; i += EX_THREADS) mloc = fmaxf(mloc, load1<DT>(tv.row, i));
    mloc = warp_max(mloc);
    s_bp[tid] = (double)mloc;
    __syncthreads();
    if (tid == 0) {
      float m = -INFINITY;
      for (int w = 0; w < EX_THREADS; w += 32) m = fmaxf(m, (float)s_bp[w]);
      s_m = m;
    }
    __syncthreads();
    if (tv.T == 0.0) {  // greedy: first argmax (sampling.py:61-64)
      int best = INT_MAX;
      for (int i = tid; i < V; i += EX_THREADS)
        if (load1<DT>(tv.row, i) == s_m) best = min(best, i);
      s_bi[tid] = best;
      __syncthreads();
      if (tid == 0) {
        int b2 = INT_MAX;
        for (int i = 0; i < EX_THREADS; ++i) b2 = min(b2, s_bi[i]);
        s_L = b2;
      }
      __syncthreads();
      for (int64_t d = tv.d0 + tid; d < tv.d1; d += EX_THREADS) {
        io.token[d] = s_L;
        if (io.flags) io.flags[d] = LC_DRAW_PRECISE;
      }
      if (tid == 0) set_kept(io, task_id, greedy_kept(V, tv.topk, tv.topp));
      __syncthreads();
      continue;
    }
    ExpCtx ec;
    ec.m = s_m;
    ec.T = tv.T;
    ec.mT = __ddiv_rn((double)s_m, tv.T);
    for (int i = tid; i < V; i += EX_THREADS) p[i] = ref_exp(ec, load1<DT>(tv.row, i));
    __syncthreads();
    {
      const double S0 = pairwise_block(p, V, s_lv, s_ls, kLeafCap, &s_bc, &s_nl);
      if (tid == 0) s_S = S0;
    }
    __syncthreads();
    for (int i = tid; i < V; i += EX_THREADS) p[i] = __ddiv_rn(p[i], s_S);
    __syncthreads();
    int L = V;
    if (tv.trunc) {
      // kept prefix of the (p desc, id asc) order.  A threshold theta on p (bisection
      // over its bit pattern, block-parallel counts/masses) selects a candidate set
      // C = {p >= theta} that surely holds the prefix (>= k elements for top-k,
      // mass >= top_p + 1e-9 for top-p); C is sorted exactly in shared memory and
      // the sequential csum of the reference runs over it.
      const int lim = tv.topk > 0 ? tv.topk : V;
      unsigned long long lo = 0ull, hi = 0x3ff0000000000001ull;  // theta in [0, 1] as bits
      // stop once C(lo) fits and holds at most ~12% more than C(hi) (which is too small)
      int cnt_lo = V, cnt_hi = 0;
      for (int it = 0; it < 64 && lo + 1 < hi && (cnt_lo > EX_CAND || cnt_lo - cnt_hi > max(64, cnt_lo >> 3));
           ++it) {
        const unsigned long long mid = lo + (hi - lo) / 2;
        const double th = __longlong_as_double((long long)mid);
        double mass = 0.0;
        int cnt = 0;
#pragma unroll 8
        for (int i = tid; i < V; i += EX_THREADS) {
          const double pi = p[i];
          if (pi >= th) {
            mass += pi;
            ++cnt;
          }
        }
        s_bp[tid] = mass;
        s_bi[tid] = cnt;
        __syncthreads();
        for (int st2 = EX_THREADS / 2; st2 > 0; st2 >>= 1) {
          if (tid < st2) {
            s_bp[tid] += s_bp[tid + st2];
            s_bi[tid] += s_bi[tid + st2];
          }
          __syncthreads();
        }
        const bool enough = tv.topk > 0 ? (s_bi[0] >= lim) : (s_bp[0] >= tv.topp + 1e-9);
        const int cmid = s_bi[0];
        __syncthreads();
        if (enough) {
          lo = mid;
          cnt_lo = cmid;
        } else {
          hi = mid;
          cnt_hi = cmid;
        }
      }
      const double theta = __longlong_as_double((long long)lo);
      // compact C (block-wide exclusive scan of per-thread counts), keys into smem
      int mycnt = 0;
      for (int i = tid; i < V; i += EX_THREADS) mycnt += (p[i] >= theta);
      s_bi[tid] = mycnt;
      __syncthreads();
      if (tid == 0) {
        int c0 = 0;
        for (int i = 0; i < EX_THREADS; ++i) {
          const int x = s_bi[i];
          s_bi[i] = c0;
          c0 += x;
        }
        s_stop = c0;
      }
      __syncthreads();
      const int nc = s_stop;
      int n = 0;
      if (nc <= EX_CAND) {
        int pos = s_bi[tid];
        for (int i = tid; i < V; i += EX_THREADS)
          if (p[i] >= theta) {
            s_key[pos] = (unsigned long long)__double_as_longlong(p[i]);
            s_id[pos] = i;
            ++pos;
          }
        int n2 = 1;
        while (n2 < nc) n2 <<= 1;
        for (int i = nc + tid; i < n2; i += EX_THREADS) {
          s_key[i] = 0ull;
          s_id[i] = INT_MAX;
        }
        __syncthreads();
        // bitonic sort: p descending, id ascending
        for (int k2 = 2; k2 <= n2; k2 <<= 1)
          for (int j2 = k2 >> 1; j2 > 0; j2 >>= 1) {
            for (int i = tid; i < n2; i += EX_THREADS) {
              const int pp = i ^ j2;
              if (pp > i) {
                const bool first_before = (s_key[i] > s_key[pp]) || (s_key[i] == s_key[pp] && s_id[i] < s_id[pp]);
                const bool desc = (i & k2) == 0;
                if (desc ? !first_before : first_before) {
                  const unsigned long long tk2 = s_key[i];
                  s_key[i] = s_key[pp];
                  s_key[pp] = tk2;
                  const int ti2 = s_id[i];
                  s_id[i] = s_id[pp];
                  s_id[pp] = ti2;
                }
              }
            }
            __syncthreads();
          }
        if (tid == 0) {
          double c = 0.0;
          int m2 = 0;
          const int lim2 = min(lim, nc);
          while (m2 < lim2) {
            ord[m2] = s_id[m2];
            ++m2;
            if (tv.topp < 1.0) {
              c += __longlong_as_double((long long)s_key[m2 - 1]);  // sequential csum (sampling.py:86)
              if (c >= tv.topp) break;
            }
          }
          s_L = m2;
        }
        __syncthreads();
        n = s_L;
      } else {
        // candidate set too large for shared memory: one block-wide argmax per element
        double last_p = INFINITY;
        int last_id = -1;
        double c = 0.0;
        while (n < lim) {
          double bp = -1.0;
          int bi = INT_MAX;
          for (int i = tid; i < V; i += EX_THREADS) {
            double pi = p[i];
            bool after = (pi < last_p) || (pi == last_p && i > last_id);
            if (after && (pi > bp || (pi == bp && i < bi))) {
              bp = pi;
              bi = i;
            }
          }
          s_bp[tid] = bp;
          s_bi[tid] = bi;
          __syncthreads();
          for (int st2 = EX_THREADS / 2; st2 > 0; st2 >>= 1) {
            if (tid < st2) {
              double op = s_bp[tid + st2];
              int oi = s_bi[tid + st2];
              if (op > s_bp[tid] || (op == s_bp[tid] && oi < s_bi[tid])) {
                s_bp[tid] = op;
                s_bi[tid] = oi;
              }
            }
            __syncthreads();
          }
          bp = s_bp[0];
          bi = s_bi[0];
          __syncthreads();
          if (bi == INT_MAX) break;
          if (tid == 0) ord[n] = bi;
          ++n;
          last_p = bp;
          last_id = bi;
          if (tv.topp < 1.0) {
            c += bp;
            if (c >= tv.topp) break;
          }
        }
      }
      L = n;
      if (tid == 0) set_kept(io, task_id, L);  // the reference's kept prefix, (p desc, id asc)
      __syncthreads();
      for (int i = tid; i < L; i += EX_THREADS) tmp[i] = p[ord[i]];
      for (int i = tid; i < V; i += EX_THREADS) q[i] = 0.0;
      __syncthreads();
      const double ks = pairwise_block(tmp, L, s_lv, s_ls, kLeafCap, &s_bc, &s_nl);
      for (int i = tid; i < L; i += EX_THREADS) q[ord[i]] = __ddiv_rn(tmp[i], ks);
    } else {
      for (int i = tid; i < V; i += EX_THREADS) q[i] = p[i];
      if (tid == 0) set_kept(io, task_id, V);
    }
    __syncthreads();
    const double Q = pairwise_block(q, V, s_lv, s_ls, kLeafCap, &s_bc, &s_nl);  // total = q.sum()
    // sample (sampling.py:97-109): numpy's cumsum(q) is sequential in id order and
    // only changes at nonzero q, so the nonzero entries are compacted in id order
    // (ord = ids, tmp = running sums), summed sequentially once, and every draw
    // binary-searches the first running sum > t
    {
      // coalesced tiles of EX_THREADS ids: ballot + per-warp offsets keep id order
      const int lane = tid & 31, wid = tid >> 5;
      int base_out = 0;
      for (int b0 = 0; b0 < V; b0 += EX_THREADS) {
        const int i = b0 + tid;
        const double qi = i < V ? q[i] : 0.0;
        const unsigned bal = __ballot_sync(0xffffffffu, qi != 0.0);
        if (lane == 0) s_bi[wid] = __popc(bal);
        __syncthreads();
        int off = base_out, tot = 0;
        for (int w = 0; w < EX_THREADS / 32; ++w) {
          const int cw = s_bi[w];
          if (w < wid) off += cw;
          tot += cw;
        }
        if (qi != 0.0) {
          const int pos = off + __popc(bal & ((1u << lane) - 1u));
          ord[pos] = i;
          tmp[pos] = qi;
        }
        base_out += tot;
        __syncthreads();
      }
      if (tid == 0) s_L = base_out;
      __syncthreads();
      // sequential running sum, staged through shared memory in kLeafCap chunks
      const int nzc = s_L;
      double c = 0.0;  // (thread 0's)
      for (int b0 = 0; b0 < nzc; b0 += kLeafCap) {
        const int nb2 = min(kLeafCap, nzc - b0);
        for (int i = tid; i < nb2; i += EX_THREADS) s_ls[i] = tmp[b0 + i];
        __syncthreads();
        if (tid == 0)
          for (int i = 0; i < nb2; ++i) {
            c += s_ls[i];
            s_ls[i] = c;
          }
        __syncthreads();
        for (int i = tid; i < nb2; i += EX_THREADS) tmp[b0 + i] = s_ls[i];
        __syncthreads();
      }
    }
    const int nz = s_L;
    for (int64_t d = tv.d0 + tid; d < tv.d1; d += EX_THREADS) {
      const double u = draw_u(io, d, tv);
      const double t = u * Q;
      int tok;
      uint8_t fl = LC_DRAW_PRECISE;
      if (!(Q > 0.0) || nz == 0) {
        tok = -1;
        fl |= LC_DRAW_BAD_ROW;
      } else {
        int lo = 0, hi = nz;  // first running sum > t
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (tmp[mid] > t) hi = mid;
          else lo = mid + 1;
        }
        double margin;
        if (lo < nz) {
          const double c = tmp[lo], prev = lo > 0 ? tmp[lo - 1] : 0.0;
          // a lower boundary of exactly 0 (no mass before) is shared with numpy exactly
          margin = fmin(prev > 0.0 ? t - prev : INFINITY, c - t);
          tok = ord[lo];
        } else {  // past the end: clamp to V - 1, back off over zeros = the last nonzero id
          margin = t - tmp[nz - 1];
          tok = ord[nz - 1];
        }
        // exp may differ from numpy's by an ulp: flag razor-thin margins
        if (margin <= fmax(t, 1e-300) * 64.0 * kEps64) {
          fl |= LC_DRAW_UNRESOLVED;
          atomicAdd(&counters[1], 1ull);
        }
      }
      io.token[d] = tok;
      if (io.flags) io.flags[d] = fl;
    }
    __syncthreads();
  }
}

// ============================== host launcher ==============================

static int g_num_sms = 0;

static int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || g_num_sms <= 0)
      g_num_sms = 148;
  }
  return g_num_sms;
}

constexpr int kExactCtas = 32;

static int grid_ctas() { return num_sms() * RS_MIN_BLOCKS; }

static int rw_cap(int64_t V) {
  const int64_t c = (V / 5 + 256 + 31) & ~31ll;
  return (int)(c < RW_NCH * 32 ? c : RW_NCH * 32);
}

int64_t workspace_bytes(int64_t n_tasks, int64_t vocab) {
  const int64_t grid = grid_ctas();
  int64_t b = 0;
  const int64_t rw_warps = (int64_t)num_sms() * 3 * RW_WARPS;
  b += ((rw_warps * rw_cap(vocab) * 16) + 3 * 255) & ~255ll;
  b += 512;
  b += ((n_tasks + 1) * 4 + 255) & ~255ll;
  b += ((n_tasks + 1) * 4 + 255) & ~255ll;
  b += ((grid * 2 * SCR_PER_CTA * 4) + 255) & ~255ll;
  b += ((grid * 2 * SCR_PER_CTA * 8) + 255) & ~255ll;
  b += ((kExactCtas * vocab * 3 * 8) + 255) & ~255ll;
  b += ((kExactCtas * vocab * 4) + 255) & ~255ll;
  b += 256;
  return b;
}

template <int DT>
static int launch_all(const char* rows, int64_t row_bytes, int V, const lc_task* tasks, int64_t n_tasks, CacheMap cm,
                      DrawIO io, void* d_ws, int64_t ws_bytes, int64_t* d_counters, cudaStream_t st) {
  if (n_tasks > INT32_MAX - 2) return LC_E_ARG;
  const int grid = grid_ctas();
  char* p = (char*)d_ws;
  auto take = [&](int64_t n) {
    char* r = p;
    p += (n + 255) & ~255ll;
    return r;
  };
  Workspace ws;
  ws.q_exact = (int*)take((n_tasks + 1) * 4);
  ws.q_cta = (int*)take((n_tasks + 1) * 4);
  ws.scr_id = (int*)take((int64_t)grid * 2 * SCR_PER_CTA * 4);
  ws.scr_e = (double*)take((int64_t)grid * 2 * SCR_PER_CTA * 8);
  const int64_t scr_stride = V;
  double* ex_scr = (double*)take(kExactCtas * scr_stride * 3 * 8);
  int32_t* ex_iscr = (int32_t*)take(kExactCtas * scr_stride * 4);
  unsigned long long* cnt = (unsigned long long*)take(64);
  RwScratch rs;
  rs.cap = rw_cap(V);
  const int64_t rw_warps = (int64_t)num_sms() * 3 * RW_WARPS;
  rs.iz = (int2*)take(rw_warps * rs.cap * 8);
  rs.e = (double*)take(rw_warps * rs.cap * 8);
  int* rw_next = (int*)take(256);
  if (!d_ws || p - (char*)d_ws > ws_bytes) {
    lcb_set_last_error("resample workspace too small (see lc_resample_workspace_bytes)", __FILE__, __LINE__);
    return LC_E_ARG;
  }
  LCB_CUDA_TRY(cudaMemsetAsync(ws.q_exact, 0, 4, st));
  LCB_CUDA_TRY(cudaMemsetAsync(ws.q_cta, 0, 4, st));
  unsigned long long* counters = d_counters ? (unsigned long long*)d_counters : cnt;
  if (!d_counters) LCB_CUDA_TRY(cudaMemsetAsync(cnt, 0, 64, st));

  const size_t smem = sizeof(Smem);
  static bool attr_set[2] = {false, false};
  if (!attr_set[DT]) {
    LCB_CUDA_TRY(cudaFuncSetAttribute(resample_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set[DT] = true;
  }
  const int rw = V <= RW_MAXV;
  // test hook: LCB_FORCE_TIER=precise|exact routes every task to that tier
  const char* ft = getenv("LCB_FORCE_TIER");
  const int force = !ft ? 0 : (ft[0] == 'p' ? 1 : (ft[0] == 'e' ? 2 : 0));
  const char* ns = getenv("LCB_NO_STAGE");
  const bool wide = force == 0 && !(ns && ns[0] == '1') && wide_eligible(DT, V, row_bytes, rows);
  if (wide) {
    // bf16 rows wider than 32000 ids: the TMA-staged top-k kernel (lc_wide.cu) takes the
    // top-k tasks and requeues everything else to the CTA kernel below
    const int rc = wide_launch(rows, row_bytes, V, tasks, n_tasks, cm, io, rw_next, ws.q_cta, counters, num_sms(), st);
    if (rc != LC_OK) return rc;
  } else if (rw && force == 0 && !(ns && ns[0] == '1') && stage_eligible(DT, V, row_bytes, rows)) {
    // bf16 rows <= 32768 ids: TMA-staged persistent kernel (lc_stage.cu); it requeues
    // what it does not handle or cannot certify to the CTA kernel below
    LCB_CUDA_TRY(cudaMemsetAsync(rw_next, 0, 4, st));
    const int rc = stage_launch(rows, row_bytes, V, tasks, n_tasks, cm, io, rw_next, ws.q_cta, counters, num_sms(), st);
    if (rc != LC_OK) return rc;
  } else if (rw) {
    // CTAs per SM: 2 (128 registers, no spills) by default; LCB_RW_BLOCKS=3 trades spills for warps
    const char* rb = getenv("LCB_RW_BLOCKS");
    const int minb = (rb && rb[0] == '3') ? 3 : RW_MIN_BLOCKS;
    const int grw = num_sms() * minb;
    const int64_t need = (n_tasks + RW_WARPS - 1) / RW_WARPS;
    const int g = (int)(need < grw ? need : grw);
    rs.next = rw_next;
    rs.q_cta = ws.q_cta;
    LCB_CUDA_TRY(cudaMemsetAsync(rw_next, 0, 4, st));
    static bool rw_attr[2][2] = {{false, false}, {false, false}};
    if (!rw_attr[DT][minb == 3]) {
      if (minb == 3)
        LCB_CUDA_TRY(cudaFuncSetAttribute(rowwarp_kernel<DT, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)sizeof(RwSmem)));
      else
        LCB_CUDA_TRY(cudaFuncSetAttribute(rowwarp_kernel<DT, RW_MIN_BLOCKS>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RwSmem)));
      rw_attr[DT][minb == 3] = true;
    }
    if (minb == 3)
      rowwarp_kernel<DT, 3><<<g, RW_THREADS, sizeof(RwSmem), st>>>(rows, row_bytes, V, tasks, (int)n_tasks, cm, io,
                                                                  ws.q_exact, counters, rs, force);
    else
      rowwarp_kernel<DT, RW_MIN_BLOCKS><<<g, RW_THREADS, sizeof(RwSmem), st>>>(rows, row_bytes, V, tasks,
                                                                              (int)n_tasks, cm, io, ws.q_exact,
                                                                              counters, rs, force);
    LCB_CUDA_TRY(cudaGetLastError());
  }
  const int g1 = (int)(n_tasks < grid ? n_tasks : grid);
  resample_kernel<DT><<<g1, RS_THREADS, smem, st>>>(rows, row_bytes, V, tasks, (int)n_tasks, cm, io, ws, counters,
                                                    (rw || wide) ? 1 : 0, force);
  LCB_CUDA_TRY(cudaGetLastError());
  static bool ex_attr[2] = {false, false};
  if (!ex_attr[DT]) {
    LCB_CUDA_TRY(cudaFuncSetAttribute(exact_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, EX_CAND * 12));
    ex_attr[DT] = true;
  }
  exact_kernel<DT><<<kExactCtas, EX_THREADS, EX_CAND * 12, st>>>(rows, row_bytes, V, tasks, ws.q_exact, cm, io, ex_scr, ex_iscr,
                                                      scr_stride, counters);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

// Optional epilogue (lc_draws.d_entropy / d_pmax): one block per task, entropy and max
// probability of softmax(z / T) over the task's row (sampling.py:112-119), fp64.
template <int DT>
__global__ void __launch_bounds__(PB_THREADS)
task_entropy_kernel(const char* rows, int64_t row_bytes, int Vdef, const lc_task* tasks, CacheMap cm, double* H,
                    double* pmax) {
  __shared__ double s_h, s_p;
  TaskView tv;
  const bool ok = resolve_task(tasks[blockIdx.x], rows, row_bytes, Vdef, cm, tv);
  if (!ok) {
    if (threadIdx.x == 0) {
      if (H) H[blockIdx.x] = nan("");
      if (pmax) pmax[blockIdx.x] = nan("");
    }
    return;
  }
  entropy_row<DT>(tv.row, tv.V, tv.T, &s_h, &s_p);
  if (threadIdx.x == 0) {
    if (H) H[blockIdx.x] = s_h;
    if (pmax) pmax[blockIdx.x] = s_p;
  }
}

int resample_launch(const void* rows, int dtype, int64_t vocab, int64_t row_stride, const lc_task* tasks,
                    int64_t n_tasks, lc_draws draws, const int32_t* pages, int max_pages, int page_rows, void* ws,
                    int64_t ws_bytes, int64_t* counters, cudaStream_t st) {
  if (n_tasks < 0 || vocab < 1 || vocab > (1 << 28) || !draws.d_token) return LC_E_ARG;
  if (!draws.d_u && !draws.d_seed) return LC_E_ARG;
  if (n_tasks == 0) return LC_OK;
  DrawIO io{draws.d_u, draws.d_seed, draws.d_index, draws.d_token, draws.d_flags, draws.d_kept};
  CacheMap cm{pages, max_pages, page_rows};
  const int64_t esz = dtype == LC_BF16 ? 2 : 4;
  int rc = LC_E_ARG;
  if (dtype == LC_BF16)
    rc = launch_all<LC_BF16>((const char*)rows, row_stride * esz, (int)vocab, tasks, n_tasks, cm, io, ws, ws_bytes,
                             counters, st);
  else if (dtype == LC_F32)
    rc = launch_all<LC_F32>((const char*)rows, row_stride * esz, (int)vocab, tasks, n_tasks, cm, io, ws, ws_bytes,
                            counters, st);
  if (rc != LC_OK || !(draws.d_entropy || draws.d_pmax)) return rc;
  for (int64_t t0 = 0; t0 < n_tasks; t0 += 65535 * 1024) {  // (grid x limit is far above; chunk for safety)
    const int64_t nt = n_tasks - t0 < 65535 * 1024 ? n_tasks - t0 : 65535 * 1024;
    if (dtype == LC_BF16)
      task_entropy_kernel<LC_BF16><<<(unsigned)nt, PB_THREADS, 0, st>>>(
          (const char*)rows, row_stride * esz, (int)vocab, tasks + t0, cm, draws.d_entropy ? draws.d_entropy + t0 : nullptr,
          draws.d_pmax ? draws.d_pmax + t0 : nullptr);
    else
      task_entropy_kernel<LC_F32><<<(unsigned)nt, PB_THREADS, 0, st>>>(
          (const char*)rows, row_stride * esz, (int)vocab, tasks + t0, cm, draws.d_entropy ? draws.d_entropy + t0 : nullptr,
          draws.d_pmax ? draws.d_pmax + t0 : nullptr);
    LCB_CUDA_TRY(cudaGetLastError());
  }
  return LC_OK;
}

}  // namespace lcb

extern "C" int64_t lc_resample_workspace_bytes(int64_t n_tasks, int64_t vocab) {
  return lcb::workspace_bytes(n_tasks, vocab);
}

extern "C" int lc_resample(const void* d_rows, int dtype, int64_t vocab, int64_t row_stride, const lc_task* d_tasks,
                           int64_t n_tasks, lc_draws draws, void* d_workspace, int64_t workspace_bytes,
                           int64_t* d_counters, void* stream) {
  if (n_tasks == 0) return LC_OK;
  if (!d_rows || !d_tasks) return LC_E_ARG;
  return lcb::resample_launch(d_rows, dtype, vocab, row_stride, d_tasks, n_tasks, draws, nullptr, 0, 1, d_workspace,
                              workspace_bytes, d_counters, (cudaStream_t)stream);
}

// Test probe: the exponentials of the FAST / PRECISE tiers, so the GPU tests
// can measure their error against fp64 and pin kEx2RelErr / kEx2Raw / kLiteErr
// (DESIGN.md "Certification").  mode 0 fast_exp, 1 cheap_exp, 2 lite_exp.
namespace lcb {
__global__ void probe_exp_kernel(const float* z, int64_t n, float m, double T, int mode, double* out) {
  __shared__ double t16[16];
  if (threadIdx.x < 16) t16[threadIdx.x] = exp2((double)threadIdx.x / 16.0);
  __syncthreads();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  ExpCtx c;
  c.m = m;
  c.T = T;
  c.mT = __ddiv_rn((double)m, T);
  double Ld = 1.4426950408889634 / T;
  c.Lhi = (float)Ld;
  c.Llo = (float)(Ld - (double)c.Lhi);
  c.md = (double)m;
  c.L16 = 16.0 * Ld;
  float a;
  if (mode == 3) {  // ex2.approx.ftz.bf16x2 of bf16(z) (the staged kernel's FAST exit test)
    const uint32_t h = f32_to_bf16_bits(z[i]);
    uint32_t r;
    asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(h | (h << 16)));
    out[i] = (double)__uint_as_float(r << 16);
    return;
  }
  out[i] = mode == 0 ? (double)fast_exp(c, z[i]) : mode == 1 ? (double)cheap_exp(c, z[i], a) : lite_exp(c, z[i], t16);
}
}  // namespace lcb

extern "C" int lc_probe_exp(const float* d_z, int64_t n, float m, double temperature, int mode, double* d_out,
                            void* stream) {
  if (n <= 0) return n == 0 ? LC_OK : LC_E_ARG;
  lcb::probe_exp_kernel<<<lcb::ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(d_z, n, m, temperature, mode, d_out);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

#ifdef LCB_RW_DEBUG
extern "C" int lcb_debug_fetch(double* out) {
  return cudaMemcpyFromSymbol(out, lcb::g_rw_dbg, sizeof(double) * 256 * 12) == cudaSuccess ? 0 : 4;
}
#endif
