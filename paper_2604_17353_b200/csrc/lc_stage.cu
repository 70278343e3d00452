// K1s: smem-staged resample kernel -- the headline regime (BASELINE configs 1-2:
// bf16 rows with V <= 32768, top-p without top-k).
//
// One persistent 512-thread CTA per SM: warp 15 produces, warps 0..14 consume.
// The producer lane fetches tasks dynamically (atomic counter), resolves them,
// publishes their metadata in shared memory and brings the row into a 3-stage
// ring of 64 KB buffers with one TMA bulk copy (cp.async.bulk + mbarrier
// complete_tx); the producer warp's lanes also precompute the task's uniforms.
// Two rows are in flight while the consumers work on the third; HBM sees every
// row exactly once, every pass after the load reads shared memory.
//
// Per row (reference semantics: sampling.py:57-109, see lc_resample.cu):
//   A  max and first argmax in one reduction (packed bf16x2 max), NaN flag.
//   B  row mass S = sum 2^((z-m)L) with fp32 MUFU exponentials, an fp64
//      accumulation and a rigorous bound (|a|-weighted).  FAST exit
//      when p(first argmax) = 1/S certainly reaches top_p: every draw is the
//      argmax (~70% of config-2 rows).
//   H  big nucleus: exact class histogram of the bf16 values that can lie above
//      the cut (z >= z_lo, with V e(z_lo) < (1-top_p) S / 2); each element's class
//      offset replaces its logit in the ring.  Class values are fp64 table
//      exponentials (<= kLiteErr), masses count x value, so the nucleus cut (class
//      b*, and how many of its ties in id order) is certified against S's bound.
//   C  per-256-id chunk kept masses from the stored class offsets; prefix.
//   D  draws: the chunk from the prefix, one warp rescans it; every decision
//      certified, otherwise the task is requeued to the CTA kernel (FAST +
//      PRECISE tiers) in lc_resample.cu.
#include "lc_common.cuh"
#include "lc_resample.cuh"
#include "lc_task.cuh"

namespace lcb {

constexpr int ST_THREADS = 512;
constexpr int ST_CW = 15;          // consumer warps (warp 15 produces)
constexpr int ST_CT = ST_CW * 32;  // consumer threads
constexpr int ST_STAGES = 3;
constexpr int ST_STAGE_BYTES = 65536;
constexpr int ST_MAXV = ST_STAGE_BYTES / 2;  // bf16
constexpr int ST_NB = 2 * ST_CT;             // histogram classes below the max (2 per consumer)
constexpr int ST_CH = 256;                   // ids per chunk (one warp x 8 per lane)
constexpr int ST_NCH = ST_MAXV / ST_CH;      // 128
constexpr int ST_NU = 32;                    // uniforms precomputed per stage (one per producer lane)
constexpr int ST_PB = 8;                     // tasks per producer grab
constexpr int ST_ND = 256;                   // draws per task handled here (more: CTA kernel)
constexpr int ST_VPT = (ST_MAXV / 8 + ST_CT - 1) / ST_CT;  // row vectors per consumer thread (9)
constexpr double kLog2e = 1.4426950408889634;
constexpr double kLn2 = 0.6931471805599453;
// ex2.approx.ftz.bf16x2 relative error incl. the bf16 rounding of its result
// (pinned by tests/test_gpu_parity.py::test_bf16_ex2_bound over every bf16 input)
constexpr float kEx2Bf16Err = 0.01f;  // measured max 0.0071 (2^-7.1)

struct __align__(128) StSmem {
  uint4 ring[ST_STAGES][ST_STAGE_BYTES / 16];
  uint32_t hist[ST_NB];
  double ev[ST_NB];        // class values e_b (valid where hist[b] > 0)
  double chm[ST_NCH];      // chunk mass of classes above the cut class
  double chp[ST_NCH + 1];  // exclusive prefix of chunk kept masses
  int chc[ST_NCH];         // chunk count of the cut class
  int chq[ST_NCH + 1];     // exclusive prefix of chc
  double su[ST_STAGES][ST_NU];  // uniforms of the stage's first draws (producer)
  double ucur[ST_NU];           // the current row's uniforms
  double dtau[ST_ND];           // big nucleus: draw targets u * K
  int dch[ST_ND];               // and their chunks
  double rd[4][ST_CW];
  float rf[ST_CW];
  int ri[2][ST_CW];
  double t16[16];
  unsigned long long full[ST_STAGES], empty[ST_STAGES];
  int stask[ST_STAGES];
  TaskView stv[ST_STAGES];  // resolved task of each stage (written by the producer)
  TaskView pbv[ST_PB];      // producer batch: resolved tasks, ids, uniforms
  int pbt[ST_PB];
  double pbu[ST_PB][ST_NU];
  double cut_e;             // cut class value
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
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
__device__ __forceinline__ uint32_t off_lo(uint32_t w) { return w & 0xffffu; }
__device__ __forceinline__ uint32_t off_hi(uint32_t w) { return w >> 16; }

// ---- consumer-group barrier (warps 0..ST_CW-1; named barrier 1) --------------------------------

__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"n"(ST_CT) : "memory"); }

__device__ __forceinline__ int st_min_i(int v, StSmem& sm, int k) {
  v = warp_min_int(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sm.ri[k][w] = v;
  cbar();
  int r = INT_MAX;
#pragma unroll
  for (int i = 0; i < ST_CW; ++i) r = min(r, sm.ri[k][i]);
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

// producer lane: fetch the next eligible task (requeueing what this kernel does
// not handle); -1 when the task list is exhausted
__device__ int st_fetch(const StageArgs& a, TaskView& tv) {
  for (;;) {
    const int t = atomicAdd(a.next, 1);
    if (t >= a.n_tasks) return -1;
    const lc_task tk = a.tasks[t];
    if (tk.draw_end <= tk.draw_begin) continue;
    const int Vt = tk.vocab > 0 ? tk.vocab : a.Vdef;
    const bool topk = tk.top_k > 0 && tk.top_k < Vt;
    const bool untrunc = !topk && tk.top_p == 1.0 && tk.temperature != 0.0;
    if (topk || untrunc || (Vt & 7) || Vt > ST_MAXV || !resolve_task(tk, a.rows, a.row_bytes, a.Vdef, a.cm, tv) ||
        (reinterpret_cast<uintptr_t>(tv.row) & 15)) {
      requeue(a, t);  // the CTA kernel handles (and reports) everything else
      continue;
    }
    return t;
  }
}

// 64-bit key: (value order, first index) -> max gives the max and its first index
__device__ __forceinline__ unsigned long long arg_key(float v, int idx) {
  return ((unsigned long long)f32_order_key(v) << 32) | (unsigned long long)(0xffffffffu - (uint32_t)idx);
}
__device__ __forceinline__ float arg_val(unsigned long long k) {
  const uint32_t o = (uint32_t)(k >> 32);
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

__global__ void __launch_bounds__(ST_THREADS, 1) stage_kernel(StageArgs a) {
  extern __shared__ __align__(128) unsigned char st_raw[];
  StSmem& sm = *reinterpret_cast<StSmem*>(st_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < ST_STAGES; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    mbar_fence_init();
  }
  if (tid < 16) sm.t16[tid] = exp2((double)tid / 16.0);
  __syncthreads();

  if (warp == ST_CW) {  // ---------------- producer warp
    // Tasks are grabbed ST_PB at a time (one atomic), loaded and resolved by parallel
    // lanes, and the first ST_NU uniforms of each computed (seed loads in parallel)
    // before the stages they go to are free; publishing is then smem stores,
    // expect_tx and one bulk copy.
    int nb = 0, bi = 0;
    bool done = false;
    for (int it = 0;; ++it) {
      const int s = it % ST_STAGES, k = it / ST_STAGES;
      while (bi == nb && !done) {  // refill the batch
        int t0 = 0;
        if (lane == 0) t0 = atomicAdd(a.next, ST_PB);
        t0 = __shfl_sync(0xffffffffu, t0, 0);
        if (t0 >= a.n_tasks) {
          done = true;
          break;
        }
        const int t = t0 + lane;
        bool ok = false;
        TaskView tv;
        if (lane < ST_PB && t < a.n_tasks) {
          const lc_task tk = a.tasks[t];
          if (tk.draw_end > tk.draw_begin) {
            const int Vt = tk.vocab > 0 ? tk.vocab : a.Vdef;
            const bool topk = tk.top_k > 0 && tk.top_k < Vt;
            const bool untrunc = !topk && tk.top_p == 1.0 && tk.temperature != 0.0;
            ok = !(topk || untrunc || (Vt & 7) || Vt > ST_MAXV) && resolve_task(tk, a.rows, a.row_bytes, a.Vdef, a.cm, tv) &&
                 !(reinterpret_cast<uintptr_t>(tv.row) & 15);
            if (!ok) requeue(a, t);  // the CTA kernel handles (and reports) everything else
          }
        }
        const unsigned okm = __ballot_sync(0xffffffffu, ok);
        if (ok) {
          const int pos = __popc(okm & ((1u << lane) - 1u));
          sm.pbt[pos] = t;
          sm.pbv[pos] = tv;
        }
        __syncwarp();
        nb = __popc(okm);
        bi = 0;
        for (int j = 0; j < nb; ++j) {
          const TaskView& tj = sm.pbv[j];
          sm.pbu[j][lane] = tj.d0 + lane < tj.d1 ? draw_u(a.io, tj.d0 + lane, tj) : 0.0;
        }
        __syncwarp();
      }
      if (lane == 0 && k > 0) mbar_wait(&sm.empty[s], (uint32_t)((k - 1) & 1));
      __syncwarp();
      if (bi == nb) {  // exhausted
        if (lane == 0) {
          sm.stask[s] = -1;
          mbar_arrive(&sm.full[s]);  // completes the phase with no bytes: consumers see -1
        }
        break;
      }
      const int j = bi++;
      sm.su[s][lane] = sm.pbu[j][lane];
      __syncwarp();
      if (lane == 0) {
        sm.stask[s] = sm.pbt[j];
        sm.stv[s] = sm.pbv[j];
        const TaskView& tj = sm.pbv[j];
        mbar_expect_tx(&sm.full[s], (uint32_t)(tj.V * 2));  // release: stask/stv/su visible
        bulk_load(sm.ring[s], tj.row, (uint32_t)(tj.V * 2), &sm.full[s]);
      }
      __syncwarp();
    }
    return;
  }

  const DrawIO& io = a.io;
  const bool prof = a.prof != nullptr && tid == 0;
  unsigned long long ph[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long tp = prof ? clock64() : 0;
#define ST_PH(k)                                \
  do {                                          \
    if (prof) {                                 \
      const unsigned long long t_ = clock64();  \
      ph[k] += t_ - tp;                         \
      tp = t_;                                  \
    }                                           \
  } while (0)
  for (int it = 0;; ++it) {  // ---------------- consumer warps
    const int s = it % ST_STAGES;
    mbar_wait(&sm.full[s], (uint32_t)((it / ST_STAGES) & 1));
    ST_PH(0);
    const int task_id = sm.stask[s];
    if (task_id < 0) break;  // fetch order is monotone: nothing after this
    const TaskView tv = sm.stv[s];
    const int V = tv.V, nvec = V >> 3;
    const int64_t d0 = tv.d0;
    const int nd = (int)(tv.d1 - tv.d0);
    // The row moves to registers: vector v = tid + ST_CT i (8 ids) is q[i] of thread
    // tid, so chunk c (256 ids = 32 vectors) is q[c / ST_CW] of warp c % ST_CW.  The
    // stage is released at once: the ring keeps three rows in flight.
    uint4 q[ST_VPT];
    {
      const uint4* R = sm.ring[s];
#pragma unroll
      for (int i = 0; i < ST_VPT; ++i) {
        const int v = tid + ST_CT * i;
        q[i] = v < nvec ? R[v] : make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u);  // -inf pad
      }
      if (tid < ST_NU) sm.ucur[tid] = sm.su[s][tid];  // the stage's uniforms outlive its release
    }
    cbar();
    if (tid == 0) mbar_arrive(&sm.empty[s]);

    // ------------------------------------------------ A: max (packed, NaN-propagating)
    uint32_t mx2 = 0xff80ff80u;
#pragma unroll
    for (int i = 0; i < ST_VPT; ++i) mx2 = bmax2_nan(mx2, bmax2_nan(bmax2_nan(q[i].x, q[i].y), bmax2_nan(q[i].z, q[i].w)));
    const float tmax = max_nan(lo_f(mx2), hi_f(mx2));
    {
      const bool tn = tmax != tmax;
      const float wm = warp_max(tn ? INFINITY : tmax);
      const bool wn = __any_sync(0xffffffffu, tn);
      if (lane == 0) {
        sm.rf[warp] = wm;
        sm.ri[0][warp] = wn;
      }
    }
    cbar();
    float m;
    bool bad;
    {
      float f8[ST_CW];
      int nb = 0;
#pragma unroll
      for (int i = 0; i < ST_CW; ++i) {
        f8[i] = sm.rf[i];
        nb |= sm.ri[0][i];
      }
#pragma unroll
      for (int w = 1; w < 16; w <<= 1)
#pragma unroll
        for (int i = 0; i + w < ST_CW; i += 2 * w) f8[i] = fmaxf(f8[i], f8[i + w]);
      m = f8[0];
      bad = nb != 0;
    }
    // (a zero maximum with both signed zeros present has a different first argmax
    // in the reference's value order: left to the CTA kernel, like non-finite rows)
    bad |= !(m > -INFINITY) || !(m < INFINITY) || m == 0.0f;
    // first argmax: only threads holding the maximum search their vectors
    auto first_argmax = [&]() -> int {
      int best = INT_MAX;
      if (tmax == m) {
#pragma unroll
        for (int i = ST_VPT - 1; i >= 0; --i) {
          const uint32_t w[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
#pragma unroll
          for (int j = 7; j >= 0; --j)
            if (((j & 1) ? hi_f(w[j >> 1]) : lo_f(w[j >> 1])) == m) best = 8 * (tid + ST_CT * i) + j;
        }
      }
      return st_min_i(best, sm, 0);
    };
    ST_PH(1);
    if (prof) ph[9]++;
    auto write_tok = [&](int tok) {
      for (int d = tid; d < nd; d += ST_CT) {
        io.token[d0 + d] = tok;
        if (io.flags) io.flags[d0 + d] = 0;
      }
    };

    bool requeue_task = false;
    if (bad) {
      requeue_task = true;  // the CTA kernel flags the row (LC_DRAW_BAD_ROW) and counts it
    } else if (tv.T == 0.0) {
      write_tok(first_argmax());
    } else {
      // ---------------------------------------------- B: FAST exit test (packed bf16x2)
      const double Ld = kLog2e / tv.T;
      const float Lf = (float)Ld;
      const float mL = fabsf(m) * Lf;
      bool fast = false;
      if (mL <= 128.0f && Lf < 1e30f) {
        const uint32_t Lb = bf16_bits(Lf);
        const float Lbf = __uint_as_float(Lb << 16);
        const uint32_t nmLb = bf16_bits(-(m * Lbf));
        const uint32_t L2 = Lb | (Lb << 16), nmL2 = nmLb | (nmLb << 16);
        float acc = 0.0f;
#pragma unroll
        for (int i = 0; i < ST_VPT; ++i) {
          acc = bacc2(acc, bex2(bfma2(q[i].x, L2, nmL2)));
          acc = bacc2(acc, bex2(bfma2(q[i].y, L2, nmL2)));
          acc = bacc2(acc, bex2(bfma2(q[i].z, L2, nmL2)));
          acc = bacc2(acc, bex2(bfma2(q[i].w, L2, nmL2)));
        }
        acc = warp_sum(acc);
        if (lane == 0) sm.rd[0][warp] = (double)acc;
        cbar();
        double Sc;
        {
          double a8[ST_CW];
#pragma unroll
          for (int i = 0; i < ST_CW; ++i) a8[i] = sm.rd[0][i];
#pragma unroll
          for (int w = 1; w < 16; w <<= 1)
#pragma unroll
            for (int i = 0; i + w < ST_CW; i += 2 * w) a8[i] += a8[i + w];
          Sc = a8[0];
        }
        const uint32_t mb = bf16_bits(m);
        const float emax = lo_f(bex2(bfma2(mb | (mb << 16), L2, nmL2)));
        // exponent error <= 2^-8 (1.001 |a| + |delta|), |delta| <= 2^-9 |m Lb|;
        // elements below 2^-40 bounded absolutely; fp32 accumulation of <= 72 terms + 32 + 15
        const float dl = 0.001953125f * mL * 1.01f + 0.001953125f;
        const double F = (double)exp2f(0.00390625f * (40.1f + dl)) * (1.0 + kEx2Bf16Err) / (1.0 - kEx2Bf16Err);
        const double tail = fmax(Sc / (double)emax - 1.0, 0.0);
        const double Sup = (1.0 + F * tail * (1.0 + 2e-5) + (double)V * 0x1p-40) * (1.0 + 1e-9);
        fast = Sup * tv.topp < 1.0 - 1e-15;
      }
      ST_PH(2);
      if (fast) {
        write_tok(first_argmax());
        ST_PH(3);
      } else {
        // -------------------------------------------- B': precise row mass (fp32 MUFU, bounded)
        // e = ex2(fl(z Lf - fl(m Lf))) / ex2(fl(m Lf - fl(m Lf))): the common rounding of m Lf
        // cancels in the ratio, the rest is |a|-weighted (W)
        const float nmL = -(m * Lf);
        const float emax = ex2_approx(fmaf(m, Lf, nmL));
        double acc = 0.0;
        float W = 0.0f;
#pragma unroll
        for (int i = 0; i < ST_VPT; ++i) {
          const uint32_t w[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
          float e8[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float z = (j & 1) ? hi_f(w[j >> 1]) : lo_f(w[j >> 1]);
            const float aa = fmaxf(fmaf(z, Lf, nmL), -200.0f);  // -inf pad -> e = 0, e*a = 0
            e8[j] = ex2_approx(aa);
            W = fmaf(e8[j], -aa, W);
          }
          acc += (double)(((e8[0] + e8[1]) + (e8[2] + e8[3])) + ((e8[4] + e8[5]) + (e8[6] + e8[7])));
        }
        {
          const double ws = warp_sum(acc), ww = warp_sum((double)W);
          if (lane == 0) {
            sm.rd[1][warp] = ws;
            sm.rd[2][warp] = ww;
          }
        }
        cbar();
        double S, Wt;
        {
          double a8[ST_CW], b8[ST_CW];
#pragma unroll
          for (int i = 0; i < ST_CW; ++i) {
            a8[i] = sm.rd[1][i];
            b8[i] = sm.rd[2][i];
          }
#pragma unroll
          for (int w = 1; w < 16; w <<= 1)
#pragma unroll
            for (int i = 0; i + w < ST_CW; i += 2 * w) {
              a8[i] += a8[i + w];
              b8[i] += b8[i + w];
            }
          S = a8[0] / (double)emax;
          Wt = b8[0] / (double)emax;
        }
        // |S - sum 2^((z-m)L)| <= ES: ex2.approx (numerator and emax), fp32 sums of 8, the
        // argument roundings (|a|-weighted: product and L; the m Lf term cancels)
        const double ES = S * (2.0 * kEx2Raw + kSum8Err + 1e-12) + Wt * 1.001 * kLn2 * 0x1p-23 +
                          S * kLn2 * 0x1p-24 * (2.0 + 0x1p-8 * (double)mL);
        const bool sane = mL <= 1e6f && Lf < 1e30f && Lf > 1e-30f && emax > 0.5f;
        // numpy's S_np vs its own e's: pairwise sum, argument rounding, libm ulps
        const double relNp = (double)(2 * V + 64) * kEps64 + 4.5e-16 * (2.0 * (double)mL + 64.0) + 2.0 * kRefExpErr;
        if (!sane) {
          requeue_task = true;
        } else {
        if (prof) ph[10]++;
        // -------------------------------------------- H: class histogram above z_lo;
        // each element's class offset replaces its logit (16 bits) in the registers
        for (int b = tid; b < ST_NB; b += ST_CT) sm.hist[b] = 0u;
        ExpCtx ec;
        ec.m = m;
        ec.T = tv.T;
        ec.Lhi = Lf;
        ec.Llo = (float)(Ld - (double)Lf);
        ec.md = (double)m;
        ec.L16 = 16.0 * Ld;
        const uint32_t km = key16(__float_as_uint(m));
        // z_lo: V e(z_lo) <= (1 - top_p) S_lo / 2, so the cut lies above it
        const double slo = fmax(S - ES, 1.0);
        const double alo = log2(fmax(0.5 * (1.0 - tv.topp) * slo / (double)V, 1e-300));
        int nb_eff = ST_NB;
        {
          const float zl = m + (float)(alo / Ld);
          if (zl > -INFINITY) nb_eff = (int)min((uint32_t)ST_NB, km - key16(__float_as_uint(zl)) + 1u);
        }
        cbar();  // hist zeroed
        // positive domain (every class in range positive): offset = bits(m) - bits(z)
        const uint32_t mb16 = __float_as_uint(m) >> 16;
        const bool pos = m > 0.0f && (uint32_t)nb_eff <= mb16 && key16_to_f(km - (uint32_t)(nb_eff - 1)) > 0.0f;
#pragma unroll
        for (int i = 0; i < ST_VPT; ++i) {
          uint32_t w[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t ol = pos ? mb16 - (w[k] & 0xffffu) : km - key16(w[k] << 16);
            const uint32_t oh = pos ? mb16 - (w[k] >> 16) : km - key16(w[k] & 0xffff0000u);
            if (ol < (uint32_t)nb_eff) atomicAdd(&sm.hist[ol], 1u);
            if (oh < (uint32_t)nb_eff) atomicAdd(&sm.hist[oh], 1u);
            w[k] = min(ol, 0xffffu) | (min(oh, 0xffffu) << 16);
          }
          q[i] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        cbar();
        ST_PH(4);
        // class values (fp64 table exp, <= kLiteErr) and masses: thread t owns classes 2t, 2t+1
        double ms[2];
        int cnt[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int b = 2 * tid + k;
          cnt[k] = (b < nb_eff) ? (int)sm.hist[b] : 0;
          ms[k] = 0.0;
          if (cnt[k] > 0) {
            const double e = lite_exp(ec, key16_to_f(km - (uint32_t)b), sm.t16);
            sm.ev[b] = e;
            ms[k] = (double)cnt[k] * e;
          }
        }
        // consumer-group exclusive scan of the class masses (descending z)
        const double tsum = ms[0] + ms[1];
        double incl = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) sm.rd[3][warp] = incl;
        cbar();
        double wpre = 0.0;
#pragma unroll
        for (int i = 0; i < ST_CW; ++i)
          if (i < warp) wpre += sm.rd[3][i];
        const double ex0 = wpre + incl - tsum;  // exclusive prefix of class 2t
        const double u53 = kEps64;
        // class values vs numpy's e: table exp + numpy's argument rounding + libm ulps
        const double relArg = 4.5e-16 * (2.0 * (double)mL + 64.0);
        const double relA = kLiteErr + kRefExpErr + relArg + (double)(ST_NB + 64) * u53;
        const double target = tv.topp * S;
        int cand = INT_MAX;
        if (ex0 + ms[0] >= target && cnt[0] > 0) cand = 2 * tid;
        else if (ex0 + ms[0] + ms[1] >= target && cnt[1] > 0) cand = 2 * tid + 1;
        const int bstar = st_min_i(cand, sm, 1);
        if (tid == 0) sm.cut_ok = 0;
        cbar();
        if (bstar != INT_MAX && (bstar >> 1) == tid) {
          const int k = bstar & 1;
          const double A = k ? ex0 + ms[0] : ex0;
          const double e = sm.ev[bstar];
          const int n = cnt[k];
          const double jd = ceil((target - A) / e);
          const int j = (int)fmin(fmax(jd, 1.0), (double)n);
          const double rho = relA + ES / S + relNp + (double)(V + 8) * u53;
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
          sm.cut_e = e;
        }
        cbar();
        ST_PH(5);
        if (!sm.cut_ok) {
          requeue_task = true;
          if (tid == 0) atomicAdd(&a.counters[4], 1ull);
        } else {
          // ------------------------------------------ C: chunk kept masses (register offsets)
          const uint32_t bs = (uint32_t)sm.cut_b;
          const int js = sm.cut_j;
          const double es = sm.cut_e;
          const int nch = (V + ST_CH - 1) / ST_CH;
#pragma unroll
          for (int i = 0; i < ST_VPT; ++i) {
            const int c = ST_CW * i + warp;
            if (c < nch) {
              const uint32_t w[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
              double msum = 0.0;
              int ccnt = 0;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const uint32_t off = (j & 1) ? off_hi(w[j >> 1]) : off_lo(w[j >> 1]);
                if (off < bs) msum += sm.ev[off];
                ccnt += (off == bs);
              }
              msum = warp_sum(msum);
              ccnt = warp_sum(ccnt);
              if (lane == 0) {
                sm.chm[c] = msum;
                sm.chc[c] = ccnt;
              }
            }
          }
          cbar();
          if (warp == 0) {
            // exclusive prefixes over chunks (4 per lane)
            int cq[4];
            double cmv[4];
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
              cmv[k] = c < nch ? sm.chm[c] + (double)takes * es : 0.0;
              if (c < nch) sm.chq[c] = cpre;
              cpre += cq[k];
              kms += cmv[k];
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
              p += cmv[k];
            }
            if (lane == 31) sm.chp[nch] = p;
          }
          if (tid == 0) sm.uncertain = 0;
          cbar();
          const double Ak = sm.chp[nch];
          // each draw's chunk (binary search over the prefix), lanes in parallel
          for (int d = tid; d < nd && d < ST_ND; d += ST_CT) {
            const double u = d < ST_NU ? sm.ucur[d] : draw_u(io, d0 + d, tv);
            const double tau = u * Ak;
            int lo = 0, hi = nch;  // first chunk whose inclusive prefix > tau
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (sm.chp[mid + 1] <= tau) lo = mid + 1;
              else hi = mid;
            }
            sm.dch[d] = lo;
            sm.dtau[d] = tau;
          }
          cbar();
          ST_PH(6);
          // ------------------------------------------ D: draws, each by its chunk's warp
          const double beta = 8.0 * kRefExpErr + kLiteErr + relArg + (double)(6 * V + 1024) * u53;
          bool unc_any = nd > ST_ND;  // (more draws than the chunk table holds: CTA kernel)
          const int ndd = min(nd, ST_ND);
          // chunk c = ST_CW i + warp lives in this warp's q[i]: each hit chunk is scanned
          // once and resolves all its draws (Best-of-N siblings crowd the argmax chunk)
#pragma unroll
          for (int i = 0; i < ST_VPT; ++i) {
            const int c = ST_CW * i + warp;
            if (c >= nch) break;
            bool any = false;
            for (int d = lane; d < ndd; d += 32) any |= sm.dch[d] == c;
            if (!__any_sync(0xffffffffu, any)) continue;
            const uint32_t w[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
            double k8[8];
            int leq = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t off = (j & 1) ? off_hi(w[j >> 1]) : off_lo(w[j >> 1]);
              k8[j] = off < bs ? sm.ev[off] : 0.0;
              leq += (off == bs);
            }
            // ranks of the cut class in id order: chunk prefix + lanes before + in-lane
            int eqi = leq;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, eqi, o);
              if (lane >= o) eqi += y;
            }
            int rank = sm.chq[c] + eqi - leq;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t off = (j & 1) ? off_hi(w[j >> 1]) : off_lo(w[j >> 1]);
              if (off == bs) {
                if (rank < js) k8[j] = es;
                ++rank;
              }
            }
            double lsum = 0.0;
#pragma unroll
            for (int j = 0; j < 8; ++j) lsum += k8[j];
            double li = lsum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const double y = __shfl_up_sync(0xffffffffu, li, o);
              if (lane >= o) li += y;
            }
            const double base = sm.chp[c] + (li - lsum);
            for (int d0b = 0; d0b < ndd; d0b += 32) {
              const int dl = d0b + lane;
              unsigned mine = __ballot_sync(0xffffffffu, dl < ndd && sm.dch[dl] == c);
              while (mine) {
                const int d = d0b + __ffs(mine) - 1;
                mine &= mine - 1;
                const double tau = sm.dtau[d];
                const unsigned hit = __ballot_sync(0xffffffffu, lsum > 0.0 && base + lsum > tau);
                bool unc = true;
                if (hit != 0) {
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
                    unc = !(Ein - tau > 2.0 * beta * Ak) || !(tau - E > 2.0 * beta * Ak) || k8[jj] == 0.0;
                    if (!unc) {
                      io.token[d0 + d] = 8 * (c * (ST_CH / 8) + lane) + jj;
                      if (io.flags) io.flags[d0 + d] = 0;
                    }
                  }
                  unc = __shfl_sync(0xffffffffu, unc, hl);
                }
                unc_any |= unc;
              }
            }
          }
          // draws whose target fell past the last chunk (rounding at u ~ 1)
          for (int d = tid; d < ndd; d += ST_CT)
            if (sm.dch[d] >= nch) unc_any = true;
          if (unc_any) sm.uncertain = 1;
          cbar();
          ST_PH(7);
          if (sm.uncertain) {
            requeue_task = true;
            if (tid == 0) atomicAdd(&a.counters[5], 1ull);
          }
          ST_PH(11);
        }
        }
      }
    }
    if (requeue_task && tid == 0) requeue(a, task_id);
    ST_PH(8);
  }
  if (prof)
    for (int k = 0; k < 12; ++k) atomicAdd(&a.prof[k], ph[k]);
#undef ST_PH
}

static unsigned long long* g_stage_prof = nullptr;

int stage_launch(const char* rows, int64_t row_bytes, int V, const lc_task* tasks, int64_t n_tasks, CacheMap cm,
                 DrawIO io, int* next, int* q_cta, unsigned long long* counters, int n_sms, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    LCB_CUDA_TRY(cudaFuncSetAttribute(stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(StSmem)));
    attr = true;
  }
  static unsigned long long* prof = nullptr;
  const char* pe = getenv("LCB_STAGE_PROF");
  if (pe && pe[0] == '1' && !prof) {
    LCB_CUDA_TRY(cudaMalloc(&prof, 16 * sizeof(unsigned long long)));
    LCB_CUDA_TRY(cudaMemset(prof, 0, 16 * sizeof(unsigned long long)));
  }
  g_stage_prof = (pe && pe[0] == '1') ? prof : nullptr;
  StageArgs a{rows, row_bytes, V, tasks, (int)n_tasks, cm, io, next, q_cta, counters, g_stage_prof};
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

// Debug: per-phase clock totals of consumer thread 0 across CTAs (LCB_STAGE_PROF=1):
// 0 wait, 1 A, 2 B, 3 fast finish, 4 H, 5 classes+cut, 6 C, 7 D, 8 end, 9 rows, 10 big rows.
// Copies and resets the counters (synchronising).
extern "C" int lcb_stage_prof_fetch(unsigned long long* h_out) {
  if (!lcb::g_stage_prof) return LC_E_ARG;
  if (cudaMemcpy(h_out, lcb::g_stage_prof, 12 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return LC_E_CUDA;
  cudaMemset(lcb::g_stage_prof, 0, 16 * sizeof(unsigned long long));
  return LC_OK;
}
