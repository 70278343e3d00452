// K1s: smem-staged resample kernel -- the headline regime (BASELINE configs 1-2:
// bf16 rows with V <= 32768, top-p without top-k).
//
// One persistent 512-thread CTA per SM.  Rows are brought into a 3-stage ring
// of 64 KB shared-memory buffers by one elected thread with TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx), tasks being fetched dynamically from
// an atomic counter at issue time, so two rows are always in flight while the
// CTA works on the third.  Every pass after the load reads shared memory only:
// HBM sees each row exactly once.
//
// Per row (reference semantics: sampling.py:57-109, see lc_resample.cu):
//   A  max / first argmax / NaN (packed bf16x2 max)
//   B  FAST exit test: row mass in packed bf16x2 arithmetic (HFMA2 + MUFU.EX2.BF16
//      at 4x the fp32 MUFU rate) with a rigorous bound; when p(first argmax)
//      certainly reaches top_p every draw is the argmax (70% of config-2 rows).
//   H  big nucleus: exact class histogram of the bf16 values within kHistOct
//      octaves of the max (shared atomics), the rest of the mass ("tail") with
//      fp32 MUFU exponentials and an error bound.  Class values are fp64
//      exponentials of numpy's own argument fl(fl(z/T) - fl(m/T)), so masses are
//      count x value: the nucleus cut (class b*, and how many of its ties in id
//      order) is certified against the combined bound.
//   C  per-256-id chunk kept masses from the class table; prefix over chunks.
//   D  draws: chunk located from the prefix, one warp rescans the chunk; every
//      decision certified, otherwise the task is requeued to the CTA kernel
//      (FAST + PRECISE tiers) in lc_resample.cu.
#include "lc_common.cuh"
#include "lc_resample.cuh"
#include "lc_task.cuh"

namespace lcb {

constexpr int ST_THREADS = 512;
constexpr int ST_WARPS = ST_THREADS / 32;
constexpr int ST_STAGES = 3;
constexpr int ST_STAGE_BYTES = 65536;
constexpr int ST_MAXV = ST_STAGE_BYTES / 2;  // bf16
constexpr int ST_NB = 1024;                  // histogram classes below the max
constexpr int ST_CH = 256;                   // ids per chunk (one warp x 8 per lane)
constexpr int ST_NCH = ST_MAXV / ST_CH;      // 128
constexpr double kHistOct = 22.0;            // histogram range, octaves of e below the max
constexpr double kLog2e = 1.4426950408889634;
// ex2.approx.ftz.bf16x2 relative error incl. the bf16 rounding of its result
// (pinned by tests/test_gpu_parity.py::test_bf16_ex2_bound over every bf16 input)
constexpr float kEx2Bf16Err = 0.01f;  // measured max 0.0071 (2^-7.1)

struct __align__(128) StSmem {
  uint4 ring[ST_STAGES][ST_STAGE_BYTES / 16];
  uint32_t hist[ST_NB];
  double ev[ST_NB];       // class values e_b (valid where hist[b] > 0)
  double chm[ST_NCH];     // chunk mass of classes above the cut class
  double chp[ST_NCH + 1]; // exclusive prefix of chunk kept masses
  int chc[ST_NCH];        // chunk count of the cut class
  int chq[ST_NCH + 1];    // exclusive prefix of chc
  double rd[2][ST_WARPS];
  float rf[ST_WARPS];
  int ri[2][ST_WARPS];
  unsigned long long mbar[ST_STAGES];
  int stask[ST_STAGES];
  double cut_A, cut_e;  // mass above the cut class, cut class value
  int cut_b, cut_j, cut_ok;
  int uncertain;
};

// ---- PTX helpers ------------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
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
__device__ __forceinline__ uint32_t bf16_bits(float f) { return (uint32_t)f32_to_bf16_bits(f); }

// ---- block reductions (512 threads) ----------------------------------------------------------

__device__ __forceinline__ double st_sum_d(double v, StSmem& sm, int k) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sm.rd[k][w] = v;
  __syncthreads();
  double r = 0.0;
#pragma unroll
  for (int i = 0; i < ST_WARPS; ++i) r += sm.rd[k][i];
  return r;
}
__device__ __forceinline__ int st_min_i(int v, StSmem& sm, int k) {
  v = warp_min_int(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sm.ri[k][w] = v;
  __syncthreads();
  int r = INT_MAX;
#pragma unroll
  for (int i = 0; i < ST_WARPS; ++i) r = min(r, sm.ri[k][i]);
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
};

__device__ __forceinline__ void requeue(const StageArgs& a, int task_id) {
  const int pos = atomicAdd(a.q_cta, 1);
  a.q_cta[1 + pos] = task_id;
}

// thread 0: fetch the next eligible task and start its row load into stage s
__device__ void st_issue(const StageArgs& a, StSmem& sm, int s) {
  for (;;) {
    const int t = atomicAdd(a.next, 1);
    if (t >= a.n_tasks) {
      sm.stask[s] = -1;
      return;
    }
    const lc_task tk = a.tasks[t];
    if (tk.draw_end <= tk.draw_begin) continue;
    TaskView tv;
    const int Vt = tk.vocab > 0 ? tk.vocab : a.Vdef;
    const bool topk = tk.top_k > 0 && tk.top_k < Vt;
    const bool untrunc = !topk && tk.top_p == 1.0 && tk.temperature != 0.0;
    if (topk || untrunc || (Vt & 7) || Vt > ST_MAXV || !resolve_task(tk, a.rows, a.row_bytes, a.Vdef, a.cm, tv) ||
        (reinterpret_cast<uintptr_t>(tv.row) & 15)) {
      requeue(a, t);  // the CTA kernel handles (and reports) everything else
      continue;
    }
    sm.stask[s] = t;
    mbar_expect_tx(&sm.mbar[s], (uint32_t)(Vt * 2));
    bulk_load(sm.ring[s], tv.row, (uint32_t)(Vt * 2), &sm.mbar[s]);
    return;
  }
}

__global__ void __launch_bounds__(ST_THREADS, 1) stage_kernel(StageArgs a) {
  extern __shared__ __align__(128) unsigned char st_raw[];
  StSmem& sm = *reinterpret_cast<StSmem*>(st_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < ST_STAGES; ++s) mbar_init(&sm.mbar[s], 1);
    mbar_fence_init();
    for (int s = 0; s < ST_STAGES; ++s) st_issue(a, sm, s);
  }
  __syncthreads();
  uint32_t phase = 0;  // bit s: parity of stage s
  for (int it = 0;; ++it) {
    const int s = it % ST_STAGES;
    const int task_id = sm.stask[s];
    if (task_id < 0) break;  // fetch order is monotone: later stages are empty too
    const lc_task tk = a.tasks[task_id];
    TaskView tv;
    resolve_task(tk, a.rows, a.row_bytes, a.Vdef, a.cm, tv);
    const int V = tv.V, nvec = V >> 3;
    mbar_wait(&sm.mbar[s], (phase >> s) & 1u);
    phase ^= 1u << s;
    const uint4* R = sm.ring[s];
    const DrawIO& io = a.io;

    // ------------------------------------------------ A: max, first argmax, NaN
    float tmax = -INFINITY;
    int tpos = -1;
    bool nan = false;
    for (int v = tid; v < nvec; v += ST_THREADS) {
      const uint4 q = R[v];
      const uint32_t x = bmax2_nan(bmax2_nan(q.x, q.y), bmax2_nan(q.z, q.w));
      const float vmax = max_nan(lo_f(x), hi_f(x));
      nan |= (vmax != vmax);
      if (vmax > tmax) {
        tmax = vmax;
        tpos = v;
      }
    }
    {
      const float wm = warp_max(tmax);
      const bool wn = __any_sync(0xffffffffu, nan);
      if (lane == 0) {
        sm.rf[warp] = wm;
        sm.ri[0][warp] = wn;
      }
    }
    __syncthreads();
    float m = -INFINITY;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < ST_WARPS; ++i) {
      m = fmaxf(m, sm.rf[i]);
      bad |= sm.ri[0][i] != 0;
    }
    __syncthreads();
    bad |= !(m > -INFINITY) || !(m < INFINITY);
    const int64_t d0 = tv.d0;
    const int nd = (int)(tv.d1 - tv.d0);
    auto write_tok = [&](int tok, uint8_t flag) {
      for (int d = tid; d < nd; d += ST_THREADS) {
        io.token[d0 + d] = tok;
        if (io.flags) io.flags[d0 + d] = flag;
      }
    };
    auto first_argmax = [&]() -> int {
      int best = INT_MAX;
      if (tpos >= 0 && tmax == m) {
        const uint4 q = R[tpos];
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int j = 7; j >= 0; --j) {
          const float f = (j & 1) ? hi_f(w[j >> 1]) : lo_f(w[j >> 1]);
          if (f == m) best = 8 * tpos + j;
        }
      }
      return st_min_i(best, sm, 0);
    };

    bool requeue_task = false;
    if (bad) {
      requeue_task = true;  // the CTA kernel flags the row (LC_DRAW_BAD_ROW) and counts it
    } else if (tv.T == 0.0) {
      const int am = first_argmax();
      write_tok(am, 0);
    } else {
      // ---------------------------------------------- B: FAST exit test (packed bf16x2)
      const double Ld = kLog2e / tv.T;
      const float Lf = (float)Ld;
      const float ml = fabsf(m) * Lf;
      bool fast = false;
      if (ml <= 128.0f && Lf < 1e30f) {
        const uint32_t Lb = bf16_bits(Lf);
        const float Lbf = __uint_as_float(Lb << 16);
        const uint32_t nmLb = bf16_bits(-(m * Lbf));
        const uint32_t L2 = Lb | (Lb << 16), nmL2 = nmLb | (nmLb << 16);
        float acc = 0.0f;
        for (int v = tid; v < nvec; v += ST_THREADS) {
          const uint4 q = R[v];
          acc = bacc2(acc, bex2(bfma2(q.x, L2, nmL2)));
          acc = bacc2(acc, bex2(bfma2(q.y, L2, nmL2)));
          acc = bacc2(acc, bex2(bfma2(q.z, L2, nmL2)));
          acc = bacc2(acc, bex2(bfma2(q.w, L2, nmL2)));
        }
        const double Sc = st_sum_d((double)acc, sm, 0);
        __syncthreads();
        const uint32_t mb = bf16_bits(m);
        const float emax = lo_f(bex2(bfma2(mb | (mb << 16), L2, nmL2)));
        // exponent error <= 2^-8 (1.001 |a| + |delta|), |delta| <= 2^-9 |m Lb|;
        // elements below 2^-40 bounded absolutely
        const float dl = 0.001953125f * ml * 1.01f + 0.001953125f;
        const double F = (double)exp2f(0.00390625f * (40.1f + dl)) * (1.0 + kEx2Bf16Err) / (1.0 - kEx2Bf16Err);
        const double tail = fmax(Sc / (double)emax - 1.0, 0.0);
        const double Sup = (1.0 + F * tail * (1.0 + 1e-5) + (double)V * 0x1p-40) * (1.0 + 1e-9);
        fast = Sup * tv.topp < 1.0 - 1e-15;
      }
      if (fast) {
        const int am = first_argmax();
        write_tok(am, 0);
      } else {
        // -------------------------------------------- H: class histogram + tail mass
        for (int b = tid; b < ST_NB; b += ST_THREADS) sm.hist[b] = 0u;
        __syncthreads();
        ExpCtx ec;
        ec.m = m;
        ec.T = tv.T;
        ec.Lhi = Lf;
        ec.Llo = (float)(Ld - (double)Lf);
        const uint32_t km = key16(__float_as_uint(m));
        int nb_eff = ST_NB;
        {
          const float zl = m - (float)(kHistOct / Ld);
          if (zl > -INFINITY) nb_eff = (int)min((uint32_t)ST_NB, km - key16(__float_as_uint(zl)) + 1u);
        }
        double tacc = 0.0;
        float W = 0.0f;
        for (int v = tid; v < nvec; v += ST_THREADS) {
          const uint4 q = R[v];
          const uint32_t w[4] = {q.x, q.y, q.z, q.w};
          float e8[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float z = (j & 1) ? hi_f(w[j >> 1]) : lo_f(w[j >> 1]);
            const uint32_t off = km - key16(__float_as_uint(z));
            float aa;
            const float e = cheap_exp(ec, z, aa);
            if (off < (uint32_t)nb_eff) {
              atomicAdd(&sm.hist[off], 1u);
              e8[j] = 0.0f;
            } else {
              e8[j] = e;
              W = fmaf(e, -aa, W);
            }
          }
          tacc += (double)(((e8[0] + e8[1]) + (e8[2] + e8[3])) + ((e8[4] + e8[5]) + (e8[6] + e8[7])));
        }
        const double tail = st_sum_d(tacc, sm, 0);
        const double Wt = st_sum_d((double)W, sm, 1) * 1.001;
        // class values and masses: thread t owns classes 2t, 2t+1
        const double mT = __ddiv_rn((double)m, tv.T);
        double ms[2];
        int cnt[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int b = 2 * tid + k;
          cnt[k] = (b < nb_eff) ? (int)sm.hist[b] : 0;
          ms[k] = 0.0;
          if (cnt[k] > 0) {
            const float z = key16_to_f(km - (uint32_t)b);
            const double e = exp(__dsub_rn(__ddiv_rn((double)z, tv.T), mT));
            sm.ev[b] = e;
            ms[k] = (double)cnt[k] * e;
          }
        }
        // block exclusive scan of the class masses (descending z)
        const double tsum = ms[0] + ms[1];
        double incl = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        __syncthreads();  // rd reads of the previous reductions are done
        if (lane == 31) sm.rd[0][warp] = incl;
        __syncthreads();
        double wpre = 0.0, Hm = 0.0;
#pragma unroll
        for (int i = 0; i < ST_WARPS; ++i) {
          const double x = sm.rd[0][i];
          if (i < warp) wpre += x;
          Hm += x;
        }
        const double ex0 = wpre + incl - tsum;  // exclusive prefix of class 2t
        const double S = Hm + tail;
        // error bound of S against numpy's sum of its own e's
        const double u53 = kEps64;
        const double relA = 2.0 * kRefExpErr + (double)(ST_NB + 64) * u53;
        const double relArgT = 2.220446049250313e-16 / tv.T;
        const double ES = Hm * relA + tail * (kEx2Raw + kSum8Err + 2.0 * kRefExpErr + 1e-12) + kArgRel * Wt +
                          relArgT * (2.0 * fabs((double)m) * tail + Wt / Ld) + S * (double)(ST_NB + 64) * u53;
        const double target = tv.topp * S;
        int cand = INT_MAX;
        if (ex0 + ms[0] >= target && cnt[0] > 0) cand = 2 * tid;
        else if (ex0 + ms[0] + ms[1] >= target && cnt[1] > 0) cand = 2 * tid + 1;
        __syncthreads();
        const int bstar = st_min_i(cand, sm, 1);
        if (tid == 0) sm.cut_ok = 0;
        __syncthreads();
        if (bstar != INT_MAX && (bstar >> 1) == tid) {
          const int k = bstar & 1;
          const double A = k ? ex0 + ms[0] : ex0;
          const double e = sm.ev[bstar];
          const int n = cnt[k];
          double jd = ceil((target - A) / e);
          int j = (int)fmin(fmax(jd, 1.0), (double)n);
          const double rho = relA + ES / S + (double)(2 * V + 64) * u53 + (double)(V + 8) * u53;
          const bool ok_hi = (A + (double)j * e) / S * (1.0 - rho) >= tv.topp;
          const bool ok_lo = (A + (double)(j - 1) * e) / S * (1.0 + rho) < tv.topp;
          // +-0 are one value for the reference (equal p, id order): a cut on a zero
          // class with the other zero class present is left to the CTA kernel
          const uint32_t kb = km - (uint32_t)bstar;
          bool zero_clash = false;
          if (kb == 0x8000u) zero_clash = bstar + 1 < nb_eff && sm.hist[bstar + 1] > 0;
          if (kb == 0x7fffu) zero_clash = bstar >= 1 && sm.hist[bstar - 1] > 0;
          sm.cut_ok = ok_hi && ok_lo && !zero_clash;
          sm.cut_b = bstar;
          sm.cut_j = j;
          sm.cut_A = A;
          sm.cut_e = e;
        }
        __syncthreads();
        if (!sm.cut_ok) {
          requeue_task = true;
          if (tid == 0) atomicAdd(&a.counters[4], 1ull);
        } else {
          // ------------------------------------------ C: chunk kept masses
          const uint32_t bs = (uint32_t)sm.cut_b;
          const int js = sm.cut_j;
          const double es = sm.cut_e;
          const int nch = (V + ST_CH - 1) / ST_CH;
          for (int c = warp; c < nch; c += ST_WARPS) {
            const int e0 = c * ST_CH + 8 * lane;
            double msum = 0.0;
            int ccnt = 0;
            if (e0 < V) {
              const uint4 q = R[e0 >> 3];
              const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float z = (j & 1) ? hi_f(w[j >> 1]) : lo_f(w[j >> 1]);
                const uint32_t off = km - key16(__float_as_uint(z));
                if (off < bs) msum += sm.ev[off];
                ccnt += (off == bs);
              }
            }
            msum = warp_sum(msum);
            ccnt = warp_sum(ccnt);
            if (lane == 0) {
              sm.chm[c] = msum;
              sm.chc[c] = ccnt;
            }
          }
          __syncthreads();
          if (warp == 0) {
            // exclusive prefixes over chunks (4 per lane)
            int cq[4];
            double cm[4];
            int cqs = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int c = lane * 4 + k;
              cq[k] = c < nch ? sm.chc[c] : 0;
              cqs += cq[k];
            }
            int cqi = cqs;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, cqi, o);
              if (lane >= o) cqi += y;
            }
            int cpre = cqi - cqs;
            double kms = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int c = lane * 4 + k;
              const int takes = min(max(js - cpre, 0), cq[k]);
              cm[k] = c < nch ? sm.chm[c] + (double)takes * es : 0.0;
              if (c < nch) sm.chq[c] = cpre;
              cpre += cq[k];
              kms += cm[k];
            }
            double kmi = kms;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const double y = __shfl_up_sync(0xffffffffu, kmi, o);
              if (lane >= o) kmi += y;
            }
            double p = kmi - kms;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int c = lane * 4 + k;
              if (c < nch) sm.chp[c] = p;
              p += cm[k];
            }
            if (lane == 31) sm.chp[nch] = p;
          }
          if (tid == 0) sm.uncertain = 0;
          __syncthreads();
          // ------------------------------------------ D: draws (one warp per draw)
          const double Ak = sm.chp[nch];
          const double beta = 8.0 * kRefExpErr + (double)(6 * V + 1024) * u53;
          for (int d = warp; d < nd; d += ST_WARPS) {
            const double u = draw_u(io, d0 + d, tv);
            const double tau = u * Ak;
            // chunk: number of chunks whose inclusive prefix <= tau
            int c = 0;
            for (int c0 = 0; c0 < nch; c0 += 32) {
              const int cc = c0 + lane;
              const bool le = cc < nch && sm.chp[cc + 1] <= tau;
              c += __popc(__ballot_sync(0xffffffffu, le));
            }
            int tok = -1;
            bool unc = false;
            if (c >= nch) {
              unc = true;
            } else {
              const int e0 = c * ST_CH + 8 * lane;
              double k8[8];
              double lsum = 0.0;
              int leq = 0;
              if (e0 < V) {
                const uint4 q = R[e0 >> 3];
                const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const float z = (j & 1) ? hi_f(w[j >> 1]) : lo_f(w[j >> 1]);
                  const uint32_t off = km - key16(__float_as_uint(z));
                  k8[j] = off < bs ? sm.ev[off] : 0.0;
                  leq += (off == bs);
                }
              } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) k8[j] = 0.0;
              }
              // ranks of the cut class in id order: chunk prefix + lanes before + in-lane
              int eqi = leq;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, eqi, o);
                if (lane >= o) eqi += y;
              }
              int rank = sm.chq[c] + eqi - leq;
              if (leq > 0 && e0 < V) {
                const uint4 q = R[e0 >> 3];
                const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const float z = (j & 1) ? hi_f(w[j >> 1]) : lo_f(w[j >> 1]);
                  if (km - key16(__float_as_uint(z)) == bs) {
                    if (rank < js) k8[j] = es;
                    ++rank;
                  }
                }
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) lsum += k8[j];
              double li = lsum;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, li, o);
                if (lane >= o) li += y;
              }
              const double base = sm.chp[c] + (li - lsum);
              const unsigned hit = __ballot_sync(0xffffffffu, lsum > 0.0 && base + lsum > tau);
              if (hit == 0) {
                unc = true;
              } else {
                const int hl = __ffs(hit) - 1;
                if (lane == hl) {
                  double E = base;
                  int jj = 0;
                  for (; jj < 8; ++jj) {
                    if (k8[jj] > 0.0 && E + k8[jj] > tau) break;
                    E += k8[jj];
                  }
                  if (jj == 8) jj = 7;  // (rounding: treated as uncertain below)
                  const double Ein = E + k8[jj];
                  tok = e0 + jj;
                  unc = !(Ein - tau > 2.0 * beta * Ak) || !(tau - E > 2.0 * beta * Ak) || k8[jj] == 0.0;
                }
                tok = __shfl_sync(0xffffffffu, tok, hl);
                unc = __shfl_sync(0xffffffffu, unc, hl);
              }
            }
            if (unc) {
              if (lane == 0) sm.uncertain = 1;
            } else if (lane == 0) {
              io.token[d0 + d] = tok;
              if (io.flags) io.flags[d0 + d] = 0;
            }
          }
          __syncthreads();
          if (sm.uncertain) {
            requeue_task = true;
            if (tid == 0) atomicAdd(&a.counters[5], 1ull);
          }
        }
      }
    }
    if (requeue_task && tid == 0) requeue(a, task_id);
    __syncthreads();  // every reader of stage s is done
    if (tid == 0) st_issue(a, sm, s);
    __syncthreads();  // stask[s] for the next round
  }
}

int stage_launch(const char* rows, int64_t row_bytes, int V, const lc_task* tasks, int64_t n_tasks, CacheMap cm,
                 DrawIO io, int* next, int* q_cta, unsigned long long* counters, int n_sms, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    LCB_CUDA_TRY(cudaFuncSetAttribute(stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(StSmem)));
    attr = true;
  }
  StageArgs a{rows, row_bytes, V, tasks, (int)n_tasks, cm, io, next, q_cta, counters};
  const int64_t g = n_tasks < n_sms ? n_tasks : n_sms;
  LCB_CUDA_TRY(cudaMemsetAsync(next, 0, 4, st));
  stage_kernel<<<(int)g, ST_THREADS, sizeof(StSmem), st>>>(a);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

bool stage_eligible(int dtype, int64_t V, int64_t row_bytes, const void* rows) {
  return dtype == LC_BF16 && V <= ST_MAXV && (V & 7) == 0 && (row_bytes & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(rows) & 15) == 0;
}

}  // namespace lcb
