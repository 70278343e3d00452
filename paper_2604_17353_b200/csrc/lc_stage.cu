// K1s: smem-staged resample kernel -- the headline regime (BASELINE configs 1-2:
// bf16 rows with V <= 32000, top-p without top-k).
//
// One persistent 512-thread CTA per SM, in three independent 5-warp groups plus a
// producer warp.  Group g owns a 64 KB shared-memory stage: it pops a resolved
// task (row pointer, parameters, its first 32 uniforms) from the producer's FIFO,
// brings the row in with one TMA bulk copy (cp.async.bulk + mbarrier complete_tx)
// and processes it with its own named barrier.  Three rows are in flight per SM
// at any time (loading or in compute), so one group's barrier and latency chains
// overlap the others' work; HBM sees every row exactly once.
//
// Per row (reference semantics: sampling.py:57-109, see lc_resample.cu):
//   A  max (packed bf16x2, NaN-propagating).
//   B  FAST exit test in packed bf16x2 arithmetic with a rigorous bound: when
//      p(first argmax) certainly reaches top_p every draw is the first argmax
//      (~70% of config-2 rows).
//   B' big nucleus: row mass S with fp32 MUFU exponentials and an |a|-weighted
//      bound; exact class histogram of the bf16 values that can lie above the cut
//      (V e(z_lo) < (1-top_p) S / 2), each element's class offset replacing its
//      logit in the stage; class values are fp64 table exponentials, masses are
//      count x value, so the cut (class b*, and how many of its ties in id order)
//      is certified against S's bound.
//   C  per-256-id chunk kept masses from the stored offsets; prefix.
//   D  draws: each hit chunk is rescanned once by one warp and resolves all its
//      draws.  Every decision is certified; an uncertain task is requeued to the
//      CTA kernel (FAST + PRECISE tiers, lc_resample.cu).
#include "lc_common.cuh"
#include "lc_resample.cuh"
#include "lc_task.cuh"
#include "lc_stage.cuh"

namespace lcb {

constexpr int SG_GROUPS = 3;
#ifndef LCB_SG_GW
#define LCB_SG_GW 5  // (6: 37.0M, 7: 36.2M rows/s vs 38.8M: spills and wider barriers)
#endif
constexpr int SG_GW = LCB_SG_GW;                // warps per group (5; -DLCB_SG_GW for experiments)
constexpr int SG_GT = SG_GW * 32;               // threads per group
constexpr int SG_PWARP = SG_GROUPS * SG_GW;     // producer warp index (15)
constexpr int SG_THREADS = (SG_PWARP + 1) * 32;  // 512
constexpr int SG_MAXV = 32000;
constexpr int SG_STAGE_BYTES = SG_MAXV * 2;
constexpr int SG_NB = 512;                       // histogram classes below the max
constexpr int SG_NU = 32;                        // uniforms precomputed per task (one per producer lane)
constexpr int SG_ND = 64;                        // draws per task handled here (more: CTA kernel)
constexpr int SG_PB = 8;                         // tasks per producer grab
constexpr int SG_FQ = 6;                         // task FIFO slots
#ifndef LCB_SG_L2PF
#define LCB_SG_L2PF 0  // (measured: 38.3M vs 38.7M rows/s with it on; TMA wait 1.9K vs 1.6K clocks)
#endif
constexpr bool SG_L2PF = LCB_SG_L2PF != 0;       // L2 prefetch of each task's row by the producer
constexpr int SG_NCK = 1;  // bulk copies per row (4, with A starting on the first quarter, measured slower: 34.8M vs 38.5M rows/s)
constexpr int SG_POPW = SG_GW - 1;               // the group warp that pops tasks (it writes no tokens for <= 128 draws)
constexpr int SG_RB = 5;                         // C: vectors per batch of independent loads
constexpr int SG_RQ = ((SG_MAXV / 8 + SG_GW * 32 - 1) / (SG_GW * 32) + 3) / 4;  // D: vectors per quarter range (7)
constexpr double kLog2e = 1.4426950408889634;
constexpr double kLn2 = 0.6931471805599453;
// ex2.approx.ftz.bf16x2 relative error incl. the bf16 rounding of its result
// (pinned by tests/test_gpu_parity.py::test_bf16_ex2_bound over every bf16 input)
constexpr float kEx2Bf16Err = 0.01f;  // measured max 0.0071 (2^-7.1)
constexpr double kEx2Bf16F = (1.0 + (double)kEx2Bf16Err) / (1.0 - (double)kEx2Bf16Err);  // ratio bound factor
// B's summation error relative to the exact sum of its (positive) bf16 exponentials: every
// exponential is added exactly-representable into fp32 (FHADD.BF16): four chains of <= 50 terms
// per thread, + 2 (the chains combined) + 5 (warp tree) additions of 2^-24 each (first order x 1.01)
constexpr double kPairAcc = 64.0 * 0x1p-24;

struct SgGroup {
  uint32_t hist[SG_NB + 32];  // + one dump bin per lane (branch-free out-of-range increments)
  double ev[SG_NB + 32];    // class values e_b (valid where hist[b] > 0); + one 0.0 per lane
  double pt[SG_GT + 1];     // C: prefix of every thread's range kept mass (+ the total)
  int tb[SG_GT];            // C: cut-class elements before every thread's range
  double su[SG_NU];         // the task's first uniforms
  double rd[3][SG_GW];
  float rf[SG_GW];
  int ri[2][SG_GW];
  TaskView tv;
  int task;
  double cut_e;
  int cut_b, cut_j, cut_ok, uncertain;
};

struct __align__(128) SgSmem {
  uint4 ring[SG_GROUPS][SG_STAGE_BYTES / 16];
  SgGroup g[SG_GROUPS];
  // producer -> groups task FIFO
  TaskView fq_tv[SG_FQ];
  int fq_task[SG_FQ];
  double fq_u[SG_FQ][SG_NU];
  int fq_tail;  // slots published (producer)
  int fq_head;  // slots claimed (groups)
  int fq_free[SG_FQ];  // per slot: the sequence number it may next be written for
  // producer batch
  TaskView pbv[SG_PB];
  int pbt[SG_PB];
  double pbu[SG_PB][SG_NU];
  double t16[16];
  unsigned long long full[SG_GROUPS][4];  // per group: one mbarrier per quarter of the row
};
static_assert(sizeof(SgSmem) <= 232448, "staged kernel shared memory");
static_assert((SG_MAXV / 8 + SG_GT - 1) / SG_GT <= 32, "argmax search: one lane per vector of a thread");

__device__ __forceinline__ void gbar(int g) { gbar_n<SG_GT>(g); }

// producer warp: grab SG_PB tasks per atomic, resolve them in parallel lanes, compute
// their first SG_NU uniforms, publish them through the FIFO; SG_GROUPS sentinels at the end
__device__ void sg_producer(const StageArgs& a, SgSmem& sm, int lane) {
  bool done = false;
  int sentinels = 0;
  // tasks per grab: SG_PB on big batches; fewer when the batch gives each group only a few rows,
  // so small launches (an engine decode step, a G = 8 rank's share) spread over every SM
  const int pb = max(1, min(SG_PB, a.n_tasks / (int)(gridDim.x * SG_GROUPS * 4)));
  for (;;) {
    int nb = 0;
    if (!done) {
      int t0 = 0;
      if (lane == 0) t0 = atomicAdd(a.next, pb);
      t0 = __shfl_sync(0xffffffffu, t0, 0);
      if (t0 >= a.n_tasks) {
        done = true;
      } else {
        const int t = t0 + lane;
        bool ok = false;
        TaskView tv;
        if (lane < pb && t < a.n_tasks) {
          const lc_task tk = a.tasks[t];
          if (tk.draw_end > tk.draw_begin) {
            const int Vt = tk.vocab > 0 ? tk.vocab : a.Vdef;
            const bool topk = tk.top_k > 0 && tk.top_k < Vt;
            const bool untrunc = !topk && tk.top_p == 1.0 && tk.temperature != 0.0;
            ok = !(topk || untrunc || (Vt & 7) || Vt > SG_MAXV) &&
                 resolve_task(tk, a.rows, a.row_bytes, a.Vdef, a.cm, tv) && !(reinterpret_cast<uintptr_t>(tv.row) & 15);
            if (!ok) requeue(a, t);  // the CTA kernel handles (and reports) everything else
          }
        }
        const unsigned okm = __ballot_sync(0xffffffffu, ok);
        if (ok) {
          const int pos = __popc(okm & ((1u << lane) - 1u));
          sm.pbt[pos] = t;
          sm.pbv[pos] = tv;
          // pull the row into L2 now: by the time a group pops the task (up to SG_FQ + SG_PB tasks
          // later) its bulk copy reads L2 instead of waiting on HBM (HBM still sees the row once)
          if (SG_L2PF) l2_prefetch(tv.row, (uint32_t)(tv.V * 2));
        }
        __syncwarp();
        nb = __popc(okm);
        // the batch's first SG_NU uniforms, all seed loads in flight together
        double ub[SG_PB];
#pragma unroll
        for (int j = 0; j < SG_PB; ++j) {
          ub[j] = 0.0;
          if (j < nb) {
            const TaskView& tj = sm.pbv[j];
            if (tj.d0 + lane < tj.d1) ub[j] = draw_u(a.io, tj.d0 + lane, tj);
          }
        }
#pragma unroll
        for (int j = 0; j < SG_PB; ++j) sm.pbu[j][lane] = ub[j];
        __syncwarp();
      }
    }
    const int npush = nb > 0 ? nb : (done ? SG_GROUPS - sentinels : 0);
    for (int j = 0; j < npush; ++j) {
      const int slot_seq = sm.fq_tail;  // (only this warp writes it)
      // wait until the slot's previous occupant (sequence slot_seq - SG_FQ) was copied out by
      // its own consumer: consumers finish out of order, so a completion count is not enough
      if (lane == 0)
        // (the FIFO is usually full: back off, so the spin takes few issue slots from the group
        // warps on this SM sub-partition; ~2 rows of look-ahead per group absorb the late wake-up)
        for (unsigned ns = 64; ld_acquire(&sm.fq_free[slot_seq % SG_FQ]) != slot_seq; ns = min(2 * ns, 1024u)) __nanosleep(ns);
      __syncwarp();
      const int slot = slot_seq % SG_FQ;
      if (nb > 0) {
        sm.fq_u[slot][lane] = sm.pbu[j][lane];
        warp_copy(sm.fq_tv[slot], sm.pbv[j], lane);
        if (lane == 0) sm.fq_task[slot] = sm.pbt[j];
      } else {
        if (lane == 0) sm.fq_task[slot] = -1;
        ++sentinels;
      }
      __syncwarp();
      if (lane == 0) st_release(&sm.fq_tail, slot_seq + 1);  // publishes the slot (cumulative release)
      __syncwarp();
    }
    if (done && sentinels >= SG_GROUPS) return;
  }
}

// group warp 0: claim the next FIFO slot, start its row load, copy the task into the group.
// The bulk copy is issued first (its complete_tx may precede the expect_tx arrive: the phase
// still needs that arrive), the arrive (release) then publishes G.task / tv / su to the group.
__device__ void sg_pop(SgSmem& sm, SgGroup& G, int g, int lane) {
  int h = 0;
  if (lane == 0) {
    h = atomicAdd(&sm.fq_head, 1);
    while (ld_acquire(&sm.fq_tail) <= h) __nanosleep(32);
  }
  h = __shfl_sync(0xffffffffu, h, 0);
  __syncwarp();  // lane 0's acquire orders the other lanes' slot reads
  const int slot = h % SG_FQ;
  const int t = sm.fq_task[slot];
  int cv = 0, nv = 0;  // vectors per chunk, per row
  if (t >= 0) {
    if (lane == 0) {
      nv = sm.fq_tv[slot].V >> 3;
      cv = (nv + SG_NCK - 1) / SG_NCK;
      const char* src = sm.fq_tv[slot].row;
      for (int c = 0; c < SG_NCK; ++c) {
        const int v0 = min(c * cv, nv), v1 = min(v0 + cv, nv);
        if (v1 > v0)
          bulk_load(sm.ring[g] + v0, src + (size_t)v0 * 16, (uint32_t)(v1 - v0) * 16u, &sm.full[g][c]);
      }
    }
    G.su[lane] = sm.fq_u[slot][lane];
    warp_copy(G.tv, sm.fq_tv[slot], lane);
  }
  __syncwarp();
  if (lane == 0) {
    G.task = t;
    st_release(&sm.fq_free[slot], h + SG_FQ);  // slot h released
    // release: G.task/tv/su visible to the group (a sentinel completes the phases with no bytes)
    for (int c = 0; c < SG_NCK; ++c) {
      const int v0 = min(c * cv, nv), v1 = min(v0 + cv, nv);
      if (v1 > v0) mbar_expect_tx(&sm.full[g][c], (uint32_t)(v1 - v0) * 16u);
      else mbar_arrive(&sm.full[g][c]);
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(SG_THREADS, 1) stage_kernel(StageArgs a) {
  extern __shared__ __align__(128) unsigned char st_raw[];
  SgSmem& sm = *reinterpret_cast<SgSmem*>(st_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < SG_GROUPS; ++s)
      for (int c = 0; c < SG_NCK; ++c) mbar_init(&sm.full[s][c], 1);
    mbar_fence_init();
    sm.fq_tail = sm.fq_head = 0;
    for (int s = 0; s < SG_FQ; ++s) sm.fq_free[s] = s;
  }
  if (tid < 16) sm.t16[tid] = exp2((double)tid / 16.0);
  if (tid < 32 * SG_GROUPS) sm.g[tid >> 5].ev[SG_NB + (tid & 31)] = 0.0;
  __syncthreads();

  if (warp == SG_PWARP) {
    sg_producer(a, sm, lane);
    return;
  }

  // (the group index broadcast from lane 0: provably warp-uniform, so the group's shared-memory
  // bases live in uniform registers and gathers / atomics address [R + UR] without an IADD)
  const int g = __shfl_sync(0xffffffffu, warp / SG_GW, 0), gw = warp % SG_GW, gt = tid - g * SG_GT;
  SgGroup& G = sm.g[g];
  // byte bases of the histogram and the class-value table: bins and (clamped) classes are
  // < 2^13, so the high half's byte offset is one shift of the packed word
  char* const hb = reinterpret_cast<char*>(G.hist);
  const char* const evb = reinterpret_cast<const char*>(G.ev);
  auto ev_at = [](const char* b, uint32_t c) { return *reinterpret_cast<const double*>(b + (lo16(c) << 3)); };
  auto ev_hi = [](const char* b, uint32_t c) { return *reinterpret_cast<const double*>(b + (c >> 13)); };
  uint4* R = sm.ring[g];
  const DrawIO& io = a.io;
  const bool prof = a.prof != nullptr && gt == 0;
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
  auto gmin_i = [&](int v, int k) -> int {
    v = warp_min_int(v);
    if (lane == 0) G.ri[k][gw] = v;
    gbar(g);
    int r = INT_MAX;
#pragma unroll
    for (int i = 0; i < SG_GW; ++i) r = min(r, G.ri[k][i]);
    return r;
  };
  auto gsum_d = [&](double v, int k) -> double {
    v = warp_sum(v);
    if (lane == 0) G.rd[k][gw] = v;
    gbar(g);
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < SG_GW; ++i) r += G.rd[k][i];
    return r;
  };

  if (gw == SG_POPW) sg_pop(sm, G, g, lane);
  for (uint32_t phase = 0;; phase ^= 1u) {
    mbar_wait(&sm.full[g][0], phase);
    ST_PH(0);
    const int task_id = G.task;
    if (task_id < 0) break;
    const TaskView tv = G.tv;
    const int V = tv.V, nvec = V >> 3;
    const int64_t d0 = tv.d0;
    const int nd = (int)(tv.d1 - tv.d0);

    // ------------------------------------------------ A: max (packed, NaN-propagating)
    // two packed running maxima per thread (3-input VHMNMX); the first argmax is searched only
    // where it is needed (FAST and greedy rows), by the threads whose maximum is the row's
    // (the row arrives in SG_NCK chunks: each chunk is waited for right before its vectors)
    uint32_t am0 = 0xff80ff80u, am1 = 0xff80ff80u;  // (-inf, -inf)
    if (SG_NCK == 1) {
#pragma unroll 5
      for (int v = gt; v < nvec; v += SG_GT) {
        const uint4 q = R[v];
        am0 = bmax2_nan(am0, bmax2_nan(q.x, q.y));
        am1 = bmax2_nan(am1, bmax2_nan(q.z, q.w));
      }
    } else {
      const int cv = (nvec + SG_NCK - 1) / SG_NCK;
      int v = gt;
      for (int c = 0; c < SG_NCK; ++c) {
        if (c > 0) mbar_wait(&sm.full[g][c], phase);
        const int v1 = min((c + 1) * cv, nvec);
#pragma unroll 4
        for (; v < v1; v += SG_GT) {
          const uint4 q = R[v];
          am0 = bmax2_nan(am0, bmax2_nan(q.x, q.y));
          am1 = bmax2_nan(am1, bmax2_nan(q.z, q.w));
        }
      }
    }
    const uint32_t amx = bmax2_nan(am0, am1);
    const float tmax = max_nan(lo_f(amx), hi_f(amx));
    const bool nan = tmax != tmax;
    {
      const float wm = warp_max(tmax);
      const bool wn = __any_sync(0xffffffffu, nan);
      if (lane == 0) {
        G.rf[gw] = wm;
        G.ri[0][gw] = wn;
      }
    }
    gbar(g);
    float m = -INFINITY;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < SG_GW; ++i) {
      m = fmaxf(m, G.rf[i]);
      bad |= G.ri[0][i] != 0;
    }
    // (a zero maximum with both signed zeros present has a different first argmax
    // in the reference's value order: left to the CTA kernel, like non-finite rows)
    bad |= !(m > -INFINITY) || !(m < INFINITY) || m == 0.0f;
    // the first argmax among this warp's "holders" (threads whose maximum is m): for each
    // holder the warp's lanes check its <= 32 vectors at once (lane k: the holder's k-th
    // vector), so the search is one round of loads + a warp min (warp-uniform result)
    auto argmax_cand = [&]() -> int {
      unsigned hm = __ballot_sync(0xffffffffu, tmax == m);
      int best = INT_MAX;
      while (hm) {
        const int th = gt - lane + (__ffs(hm) - 1);
        hm &= hm - 1;
        const int v = th + lane * SG_GT;
        int pos = INT_MAX;
        if (v < nvec) {
          const uint4 q = R[v];
          const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int j = 7; j >= 0; --j)
            if (((j & 1) ? hi_f(w[j >> 1]) : lo_f(w[j >> 1])) == m) pos = 8 * v + j;
        }
        best = min(best, warp_min_int(pos));
      }
      return best;
    };
    auto first_argmax = [&]() -> int { return gmin_i(argmax_cand(), 1); };
    ST_PH(1);
    if (prof) ph[9]++;
    auto write_tok = [&](int tok) {
      for (int d = gt; d < nd; d += SG_GT) {
        io.token[d0 + d] = tok;
        if (io.flags) io.flags[d0 + d] = 0;
      }
    };

    bool requeue_task = false;
    bool popped = false;  // the next task was popped (and its row load issued) early
    if (bad) {
      requeue_task = true;  // the CTA kernel flags the row (LC_DRAW_BAD_ROW) and counts it
    } else if (tv.T == 0.0) {
      write_tok(first_argmax());
      if (gt == 0) set_kept(io, task_id, greedy_kept(V, tv.topk, tv.topp));
    } else {
      // ---------------------------------------------- B: FAST exit test (packed bf16x2)
      const double Ld = tv.Ld;  // = kLog2e / tv.T, divided once by the producer
      const float Lf = (float)Ld;
      const float mL = fabsf(m) * Lf;
      bool fast = false;
      double Sfast = 1.0;  // FAST estimate of the row mass (within its bound factor)
      int amax = INT_MAX;  // first argmax (set with the FAST mass)
      if (mL <= 128.0f && Lf < 1e30f) {
        const uint32_t Lb = bf16_bits(Lf);
        const float Lbf = __uint_as_float(Lb << 16);
        const uint32_t nmLb = bf16_bits(-(m * Lbf));
        const uint32_t L2 = Lb | (Lb << 16), nmL2 = nmLb | (nmLb << 16);
        // the 8 bf16 exponentials of a vector are added straight into four fp32 chains (one per
        // word: <= 50 terms each)
        float ac0 = 0.0f, ac1 = 0.0f, ac2 = 0.0f, ac3 = 0.0f;
#pragma unroll 4
        for (int v = gt; v < nvec; v += SG_GT) {
          const uint4 q = R[v];
          ac0 = bex2_acc(ac0, bfma2(q.x, L2, nmL2));
          ac1 = bex2_acc(ac1, bfma2(q.y, L2, nmL2));
          ac2 = bex2_acc(ac2, bfma2(q.z, L2, nmL2));
          ac3 = bex2_acc(ac3, bfma2(q.w, L2, nmL2));
        }
        const float acc = (ac0 + ac1) + (ac2 + ac3);
        // one barrier for the mass and the first argmax
        {
          const float ws = warp_sum(acc);
          const int wc = argmax_cand();
          if (lane == 0) {
            G.rd[0][gw] = (double)ws;
            G.ri[1][gw] = wc;
          }
        }
        gbar(g);
        double Sc = 0.0;
#pragma unroll
        for (int i = 0; i < SG_GW; ++i) {
          Sc += G.rd[0][i];
          amax = min(amax, G.ri[1][i]);
        }
        const uint32_t mb = bf16_bits(m);
        const float emax = lo_f(bex2(bfma2(mb | (mb << 16), L2, nmL2)));
        // exponent error <= 2^-8 (1.001 |a| + |delta|), |delta| <= 2^-9 |m Lb|;
        // elements below 2^-40 bounded absolutely.  Summation: Sc <= (1 + kPairAcc) sum E_i
        // (fp32 chains of <= 50 + 2 + 5 terms, all positive), so
        // sum_{i != amax} E_i / E_max <= Sc (1 + kPairAcc) / E_max - 1
        const float dl = 0.001953125f * mL * 1.01f + 0.001953125f;
        // (no fp64 divisions on this per-row path: the ratio is a constant, 1/emax a correctly
        // rounded reciprocal -- one extra 2^-53 rounding, far inside the 1e-9 / V 2^-40 slack)
        const double F = (double)exp2f(0.00390625f * (40.1f + dl)) * kEx2Bf16F;
        const double tail = fmax(Sc * (1.0 + kPairAcc) * __drcp_rn((double)emax) - 1.0, 0.0);
        Sfast = 1.0 + tail;
        const double Sup = (1.0 + F * tail + (double)V * 0x1p-40) * (1.0 + 1e-9);
        fast = Sup * tv.topp < 1.0 - 1e-15;
      }
      ST_PH(2);
      if (fast) {
        // the stage is free (only m and amax are needed now): start the next row's load while
        // the tokens are written
        ST_PH(2);
        if (gw == SG_POPW) sg_pop(sm, G, g, lane);
        ST_PH(11);
        popped = true;
        write_tok(amax);
        if (gt == 0) set_kept(io, task_id, 1);
        ST_PH(3);
      } else {
        if (prof) ph[10]++;
        // -------------------------------------------- H: one pass over the row: exact class
        // histogram of the values that can lie above the cut (z >= z_lo, with V e(z_lo) <=
        // (1 - top_p) S / 2), fp32 MUFU exponentials for the rest (the "tail", bounded), and
        // every element's class offset written over its logit (16 bits) in the stage
        for (int b = gt; b < SG_NB; b += SG_GT) G.hist[b] = 0u;
        ExpCtx ec;
        ec.m = m;
        ec.T = tv.T;
        ec.Lhi = Lf;
        ec.Llo = (float)(Ld - (double)Lf);
        ec.md = (double)m;
        ec.L16 = 16.0 * Ld;
        const uint32_t km = key16(__float_as_uint(m));
        // the exact histogram spans the SG_NB classes (bf16 values) below the max: every value
        // there is counted exactly, everything further down is the "tail" (a cut outside the
        // histogram is detected and requeued).  A fixed span lets one packed min clamp every
        // offset >= SG_NB onto the lane's dump bin.
        const int nb_eff = SG_NB;
        // e = ex2(fl(z Lf - fl(m Lf))) / ex2(fl(m Lf - fl(m Lf))): the common rounding of m Lf
        // cancels in the ratio, the rest weighs |a|
        const float nmL = -(m * Lf);
        const float emax = ex2_approx(fmaf(m, Lf, nmL));
        const bool sane = mL <= 1e6f && Lf < 1e30f && Lf > 1e-30f && emax > 0.5f;
        // positive domain (every class in range positive): offset = bits(m) - bits(z)
        const uint32_t mb16 = __float_as_uint(m) >> 16;
        const bool pos = m > 0.0f && (uint32_t)nb_eff <= mb16 && key16_to_f(km - (uint32_t)(nb_eff - 1)) > 0.0f;
        gbar(g);  // hist zeroed
        double tacc = 0.0;
        if (pos) {
          // offsets of both halves at once: bits(m) - bits(z) per 16-bit lane (VIADD.16x2);
          // negative z wrap to >= bits(m) + 1 > nb_eff, never a kept class
          const uint32_t mb2 = (mb16 | (mb16 << 16)) + 0x00010001u;
          const uint32_t dump2 = (uint32_t)(SG_NB + lane) * 0x00010001u;
          #pragma unroll 4
          for (int v = gt; v < nvec; v += SG_GT) {
            const uint4 q = R[v];
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
            uint32_t o[4];
            float2 e2[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              o[k] = __vadd2(~w[k], mb2);
              // histogram bins: offsets clamped (one packed min) to the lane's dump bin; bins in
              // [nb_eff, SG_NB) also count tail elements and are never read
              const uint32_t hc = __vminu2(o[k], dump2);
              // (both bins < 2^14: the high bin's byte offset is hc >> 14, one LEA.HI)
              atomicAdd(reinterpret_cast<uint32_t*>(hb + (lo16(hc) << 2)), 1u);
              atomicAdd(reinterpret_cast<uint32_t*>(hb + (hc >> 14)), 1u);
              const uint32_t ol = o[k] & 0xffffu, oh = o[k] >> 16;
              const bool il = ol < (uint32_t)nb_eff, ih = oh < (uint32_t)nb_eff;
              // both halves' arguments in one FFMA2; -inf -> 0
              const float2 x = ffma2_rn(make_float2(lo_f(w[k]), hi_f(w[k])), Lf, nmL);
              e2[k] = make_float2(il ? 0.0f : ex2_approx(x.x), ih ? 0.0f : ex2_approx(x.y));
            }
            // balanced 3-level fp32 tree over the 8 (kSum8Err) in packed FADD2
            const float2 s2 = fadd2_rn(fadd2_rn(e2[0], e2[1]), fadd2_rn(e2[2], e2[3]));
            tacc += (double)(s2.x + s2.y);
            R[v] = make_uint4(o[0], o[1], o[2], o[3]);
          }
        } else {
          #pragma unroll 4
          for (int v = gt; v < nvec; v += SG_GT) {
            const uint4 q = R[v];
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
            uint32_t o[4];
            float2 e2[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t ol = km - key16(w[k] << 16), oh = km - key16(w[k] & 0xffff0000u);
              const bool il = ol < (uint32_t)nb_eff, ih = oh < (uint32_t)nb_eff;
              atomicAdd(&G.hist[min(ol, (uint32_t)(SG_NB + lane))], 1u);
              atomicAdd(&G.hist[min(oh, (uint32_t)(SG_NB + lane))], 1u);
              const float2 x = ffma2_rn(make_float2(lo_f(w[k]), hi_f(w[k])), Lf, nmL);
              e2[k] = make_float2(il ? 0.0f : ex2_approx(x.x), ih ? 0.0f : ex2_approx(x.y));
              o[k] = ol | (oh << 16);
            }
            const float2 s2 = fadd2_rn(fadd2_rn(e2[0], e2[1]), fadd2_rn(e2[2], e2[3]));
            tacc += (double)(s2.x + s2.y);
            R[v] = make_uint4(o[0], o[1], o[2], o[3]);
          }
        }
        const double tail = gsum_d(tacc, 1) * __drcp_rn((double)emax);  // (2^-53 inside the 1e-12 slack)
        // numpy's S_np vs its own e's: pairwise sum, argument rounding, libm ulps
        const double relNp = (double)(2 * V + 64) * kEps64 + 4.5e-16 * (2.0 * (double)mL + 64.0) + 2.0 * kRefExpErr;
        if (!sane) {
          requeue_task = true;
        } else {
          ST_PH(4);
          // class values (fp64 table exp, <= kLiteErr) and masses: thread owns classes
          // SGC*gt .. SGC*gt + SGC-1
          constexpr int SGC = SG_NB / SG_GT + (SG_NB % SG_GT ? 1 : 0);  // 4
          double ms[SGC];
          int cnt[SGC];
          double tsum = 0.0;
#pragma unroll
          for (int k = 0; k < SGC; ++k) {
            const int b = SGC * gt + k;
            cnt[k] = (b < nb_eff) ? (int)G.hist[b] : 0;
            ms[k] = 0.0;
            if (cnt[k] > 0) {
              const double e = lite_exp(ec, key16_to_f(km - (uint32_t)b), sm.t16);
              G.ev[b] = e;
              ms[k] = (double)cnt[k] * e;
            }
            tsum += ms[k];
          }
          // group exclusive scan of the class masses (descending z)
          double incl = tsum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          if (lane == 31) G.rd[0][gw] = incl;
          gbar(g);
          double wpre = 0.0, Hm = 0.0;
#pragma unroll
          for (int i = 0; i < SG_GW; ++i) {
            if (i < gw) wpre += G.rd[0][i];
            Hm += G.rd[0][i];
          }
          const double u53 = kEps64;
          const double S = Hm + tail;
          // class values vs numpy's e: table exp + numpy's argument rounding + libm ulps
          const double relArg = 4.5e-16 * (2.0 * (double)mL + 64.0);
          const double relA = kLiteErr + kRefExpErr + relArg + (double)(SG_NB + 64) * u53;
          // |S - sum e| <= ES: classes (relA), tail: ex2.approx (numerator and emax), fp32
          // sums of 8, the argument roundings (|a|-weighted; the m Lf term cancels)
          // (tail arguments |a| <= 2^8 |m L| + 130: an element below -126 octaves flushes to 0
          // and is bounded by V 2^-126; the rounding of a weighs |a| ln2 2^-23)
          const double amax_t = 130.0 + (double)mL;
          double Scut = S;
          double EScut = Hm * relA + tail * (2.0 * kEx2Raw + kSum8Err + 1e-12 + amax_t * kLn2 * 0x1p-23) +
                         (double)V * 0x1p-126 + S * 64.0 * u53;
          int bstar = INT_MAX;
          int cut_ok = 0;
          for (int pass = 0; pass < 2; ++pass) {
            if (pass == 1) {
              // PRECISE tail (rare: the FAST tail's bound left the cut undecided): every tail
              // element's logit is recovered from its stored offset (both encodings are
              // 16-bit bijections) and its fp64 table exponential summed
              double tp2 = 0.0;
              for (int v = gt; v < nvec; v += SG_GT) {
                const uint4 q = R[v];
                const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const uint32_t off = (j & 1) ? off_hi(w[j >> 1]) : off_lo(w[j >> 1]);
                  if (off >= (uint32_t)nb_eff) {
                    const float z = pos ? __uint_as_float(((mb16 - off) & 0xffffu) << 16)
                                        : key16_to_f((km - off) & 0xffffu);
                    tp2 += lite_exp(ec, z, sm.t16);
                  }
                }
              }
              const double tailp = gsum_d(tp2, 2);
              Scut = Hm + tailp;
              EScut = (Hm + tailp) * relA + (double)V * 0x1p-126 + Scut * (double)(V + 64) * u53;
            }
            const double target = tv.topp * Scut;
            int cand = INT_MAX;
            {
              double ex = wpre + incl - tsum;
#pragma unroll
              for (int k = 0; k < SGC; ++k) {
                if (cand == INT_MAX && cnt[k] > 0 && ex + ms[k] >= target) cand = SGC * gt + k;
                ex += ms[k];
              }
            }
            bstar = gmin_i(cand, 0);
            if (bstar == INT_MAX) break;  // (uniform) no cut class in the histogram range
            if (bstar / SGC == gt) {  // the owner of the cut class decides (0 uncertain, 1 ok, 2 +-0)
              double A = wpre + incl - tsum;
              int n = 0;
#pragma unroll
              for (int k = 0; k < SGC; ++k) {
                if (SGC * gt + k < bstar) A += ms[k];
                if (SGC * gt + k == bstar) n = cnt[k];
              }
              const double e = G.ev[bstar];
              // (no fp64 divisions on this serial path: correctly rounded reciprocals, one more
              // rounding per quotient inside rho's slack; j only proposes the tie count, the two
              // certified inequalities decide it)
              const double rS = __drcp_rn(Scut);
              const double jd = ceil((target - A) * __drcp_rn(e));
              const int j = (int)fmin(fmax(jd, 1.0), (double)n);
              const double rho = relA + EScut * rS * (1.0 + 4.0 * u53) + relNp + (double)(V + 12) * u53;
              const bool ok_hi = (A + (double)j * e) * rS * (1.0 - rho) >= tv.topp;
              const bool ok_lo = (A + (double)(j - 1) * e) * rS * (1.0 + rho) < tv.topp;
              // +-0 are one value for the reference (equal p, id order): a cut on a zero
              // class with the other zero class present is left to the CTA kernel
              const uint32_t kb = km - (uint32_t)bstar;
              bool zero_clash = false;
              if (kb == 0x8000u) zero_clash = bstar + 1 < nb_eff && G.hist[bstar + 1] > 0;
              if (kb == 0x7fffu) zero_clash = bstar >= 1 && G.hist[bstar - 1] > 0;
              const int ok = zero_clash ? 2 : (ok_hi && ok_lo);
              G.cut_ok = ok;
              G.cut_b = bstar;
              G.cut_j = j;
              G.cut_e = e;
              // the cut class's table entry is zeroed: C and D clamp every offset >= bs onto
              // it (its value stays in G.cut_e)
              if (ok == 1) G.ev[bstar] = 0.0;
            }
            gbar(g);
            cut_ok = G.cut_ok;
            if (cut_ok != 0) break;
            if (pass == 0 && gt == 0) atomicAdd(&a.counters[7], 1ull);  // precise tails computed
          }
          ST_PH(5);
          if (cut_ok != 1) {
            requeue_task = true;
            // counters: 4 cut not certified (even with the precise tail), 6 no cut class in the
            // histogram range (or a +-0 cut); 7 counts precise-tail recomputations
            if (gt == 0) atomicAdd(&a.counters[(bstar == INT_MAX || cut_ok == 2) ? 6 : 4], 1ull);
          } else {
            // ---------------------------------------- C: every thread sums the kept mass of its
            // own contiguous range of Rv vectors (classes above the cut class, fp64 values
            // gathered for kept elements only, plus a count of the cut class); one group scan
            // turns the ranges into prefixes P_t (tie ranks: the first js cut-class elements
            // in id order are kept, so the ties before range t contribute min(js, tb_t) es)
            const uint32_t bs = (uint32_t)G.cut_b;
            const uint32_t bs2 = bs | (bs << 16);
            const int js = G.cut_j;
            const double es = G.cut_e;
            const int Rv = (nvec + SG_GT - 1) / SG_GT;  // vectors per range (25 at V = 32000)
            const int v0 = min(Rv * gt, nvec), v1 = min(v0 + Rv, nvec);
            double ma = 0.0;
            // cut-class elements counted packed: per 16-bit half, 1 unless the offset is bs
            // (xor + one packed min), subtracted from the number of halves visited
            uint32_t ne2 = 0u;
            int nvis = 0;
            for (int vb = v0; vb < v1; vb += SG_RB) {
              nvis += SG_RB;
              uint32_t w[SG_RB][4];
#pragma unroll
              for (int k = 0; k < SG_RB; ++k) {
                uint4 q = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                if (vb + k < v1) q = R[vb + k];
                w[k][0] = q.x;
                w[k][1] = q.y;
                w[k][2] = q.z;
                w[k][3] = q.w;
              }
              double a0 = 0.0, a1 = 0.0;
#pragma unroll
              for (int k = 0; k < SG_RB; ++k) {
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  // offsets >= bs clamped (one packed min) onto the zeroed entry bs
                  const uint32_t c = __vminu2(w[k][h], bs2);
                  a0 += ev_at(evb, c);
                  a1 += ev_hi(evb, c);
                  ne2 += __vminu2(w[k][h] ^ bs2, 0x00010001u);
                }
              }
              ma += a0 + a1;
            }
            const int mc = 8 * nvis - (int)((ne2 & 0xffffu) + (ne2 >> 16));
            // group inclusive scan of (ma, mc)
            double mi = ma;
            int ci = mc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const double y = __shfl_up_sync(0xffffffffu, mi, o);
              const int z = __shfl_up_sync(0xffffffffu, ci, o);
              if (lane >= o) {
                mi += y;
                ci += z;
              }
            }
            if (lane == 31) {
              G.rd[2][gw] = mi;
              G.ri[1][gw] = ci;
            }
            if (gt == 0) G.uncertain = 0;
            gbar(g);
            double mw = 0.0, mtot = 0.0;
            int cw = 0, ctot = 0;
#pragma unroll
            for (int i = 0; i < SG_GW; ++i) {
              if (i < gw) {
                mw += G.rd[2][i];
                cw += G.ri[1][i];
              }
              mtot += G.rd[2][i];
              ctot += G.ri[1][i];
            }
            {
              const int tb = cw + ci - mc;  // cut-class elements before this range
              G.pt[gt] = (mw + mi - ma) + (double)min(js, tb) * es;
              G.tb[gt] = tb;
              if (gt == 0) G.pt[SG_GT] = mtot + (double)min(js, ctot) * es;
            }
            gbar(g);
            const double Ak = G.pt[SG_GT];
            const int ndd = min(nd, SG_ND);
            ST_PH(6);
            // ---------------------------------------- D: a quad of lanes per draw.  Every lane
            // finds the range holding the draw's target (binary search over the prefixes), takes
            // a quarter of that range's vectors (independent loads, per-vector kept masses kept in
            // registers), the quad scans its quarters, and the lane whose quarter holds the target
            // walks its vectors and then the hit vector's 8 elements
            const double beta = 8.0 * kRefExpErr + kLiteErr + relArg + (double)(6 * V + 1024) * u53;
            bool unc_any = nd > SG_ND;  // (more draws than handled here: CTA kernel)
            const int Rq = (Rv + 3) >> 2;  // vectors per quarter (<= SG_RQ)
            const int q = lane & 3;
            for (int db = 0; db < ndd; db += SG_GT / 4) {
              const int d = db + (gt >> 2);
              const bool act = d < ndd;
              double tau = 0.0;
              if (act) tau = (d < SG_NU ? G.su[d] : draw_u(io, d0 + d, tv)) * Ak;
              int t = 0;  // the last range whose prefix is <= tau
#pragma unroll
              for (int st = 128; st > 0; st >>= 1)
                if (t + st < SG_GT && G.pt[t + st] <= tau) t += st;
              const int w0 = min(Rv * t, nvec), w1 = min(w0 + Rv, nvec);
              const int x0 = min(w0 + Rq * q, w1), x1 = min(x0 + Rq, w1);
              double mk[SG_RQ];
              int tk[SG_RQ];
              double ma_q = 0.0;
              int c_q = 0;
#pragma unroll
              for (int k = 0; k < SG_RQ; ++k) {
                uint4 qv = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                if (act && x0 + k < x1) qv = R[x0 + k];
                const uint32_t w[4] = {qv.x, qv.y, qv.z, qv.w};
                double a0 = 0.0, a1 = 0.0;
                uint32_t n2 = 0u;  // packed: halves whose offset is not bs
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  const uint32_t cl = __vminu2(w[h], bs2);
                  a0 += ev_at(evb, cl);
                  a1 += ev_hi(evb, cl);
                  n2 += __vminu2(w[h] ^ bs2, 0x00010001u);
                }
                const int c = 8 - (int)((n2 & 0xffffu) + (n2 >> 16));
                mk[k] = a0 + a1;
                tk[k] = c;
                ma_q += mk[k];
                c_q += c;
              }
              // exclusive scan of (ma, c) over the quad
              double ea = ma_q;
              int ec = c_q;
#pragma unroll
              for (int o = 1; o < 4; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, ea, o, 4);
                const int z = __shfl_up_sync(0xffffffffu, ec, o, 4);
                if (q >= o) {
                  ea += y;
                  ec += z;
                }
              }
              ea -= ma_q;
              ec -= c_q;
              const int tb0 = G.tb[t];
              int rank = tb0 + ec;  // cut-class elements before this quarter
              double E = G.pt[t] + ea + (double)(min(js, rank) - min(js, tb0)) * es;
              const double Eend = E + ma_q + (double)(min(js, rank + c_q) - min(js, rank)) * es;
              const bool mine = act && E <= tau && tau < Eend;
              const unsigned qm = (__ballot_sync(0xffffffffu, mine) >> (lane & ~3)) & 0xfu;
              bool unc = act && (qm == 0u || !(tau < Ak));  // (rounding at a range end, u ~ 1)
              if (mine && !unc) {
                int hv = -1;
#pragma unroll
                for (int k = 0; k < SG_RQ; ++k) {
                  if (hv < 0 && x0 + k < x1) {
                    const double m_k = mk[k] + (double)(min(js, rank + tk[k]) - min(js, rank)) * es;
                    if (E + m_k > tau) {
                      hv = x0 + k;
                    } else {
                      E += m_k;
                      rank += tk[k];
                    }
                  }
                }
                unc = true;
                if (hv >= 0) {
                  const uint4 hq = R[hv];
                  const uint32_t hw[4] = {hq.x, hq.y, hq.z, hq.w};
                  int jj = 0;
                  double kk = 0.0;
                  for (; jj < 8; ++jj) {
                    const uint32_t off = (jj & 1) ? off_hi(hw[jj >> 1]) : off_lo(hw[jj >> 1]);
                    kk = off < bs ? G.ev[off] : 0.0;
                    if (off == bs) kk = (rank++ < js) ? es : 0.0;
                    if (kk > 0.0 && E + kk > tau) break;
                    E += kk;
                  }
                  if (jj < 8) {
                    const double Ein = E + kk;
                    unc = !(Ein - tau > 2.0 * beta * Ak) || !(tau - E > 2.0 * beta * Ak);
                    if (!unc) {
                      io.token[d0 + d] = 8 * hv + jj;
                      if (io.flags) io.flags[d0 + d] = 0;
                    }
                  }
                }
              }
              unc_any |= unc;
            }
            if (unc_any) G.uncertain = 1;
            gbar(g);
            // the stage is free: the next row's load overlaps the kept count and the requeue
            ST_PH(7);
            if (gw == SG_POPW) sg_pop(sm, G, g, lane);
            ST_PH(11);
            popped = true;
            if (G.uncertain) {
              requeue_task = true;
              if (gt == 0) atomicAdd(&a.counters[5], 1ull);
            } else if (io.kept && gw == 0) {
              // |kept| = every class above the cut class + its first js ties in id order
              int kc = 0;
              for (int b = lane; b < (int)bs; b += 32) kc += (int)G.hist[b];
              kc = warp_sum(kc);
              if (lane == 0) io.kept[task_id] = kc + js;
            }
          }
        }
      }
    }
    if (requeue_task && gt == 0) requeue(a, task_id);
    gbar(g);  // the group is done with its stage
    ST_PH(8);
    if (gw == SG_POPW && !popped) sg_pop(sm, G, g, lane);
    ST_PH(11);
  }
  if (prof)
    for (int k = 0; k < 12; ++k) atomicAdd(&a.prof[k], ph[k]);
#undef ST_PH
}

static unsigned long long* g_stage_prof = nullptr;

// the LCB_STAGE_PROF buffer (nullptr when profiling is off), shared with lc_wide.cu
unsigned long long* stage_prof_buffer() {
  static unsigned long long* prof = nullptr;
  const char* pe = getenv("LCB_STAGE_PROF");
  if (!(pe && pe[0] == '1')) return nullptr;
  if (!prof && cudaMalloc(&prof, 16 * sizeof(unsigned long long)) == cudaSuccess)
    cudaMemset(prof, 0, 16 * sizeof(unsigned long long));
  g_stage_prof = prof;
  return prof;
}

int stage_launch(const char* rows, int64_t row_bytes, int V, const lc_task* tasks, int64_t n_tasks, CacheMap cm,
                 DrawIO io, int* next, int* q_cta, unsigned long long* counters, int n_sms, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    LCB_CUDA_TRY(cudaFuncSetAttribute(stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SgSmem)));
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
  stage_kernel<<<(int)g, SG_THREADS, sizeof(SgSmem), st>>>(a);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

bool stage_eligible(int dtype, int64_t V, int64_t row_bytes, const void* rows) {
  return dtype == LC_BF16 && V <= SG_MAXV && (V & 7) == 0 && (row_bytes & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(rows) & 15) == 0;
}

}  // namespace lcb

// Debug: per-phase clock totals of each group's thread 0 across CTAs (LCB_STAGE_PROF=1):
// 0 wait, 1 A, 2 B, 3 fast finish, 4 B'+H, 5 classes+cut, 6 C, 7 D, 8 end, 9 rows, 10 big rows,
// 11 task pops (group warp 0: FIFO claim, task copy, row load issue).
// Copies and resets the counters (synchronising).
extern "C" int lcb_stage_prof_fetch(unsigned long long* h_out) {
  if (!lcb::g_stage_prof) return LC_E_ARG;
  if (cudaMemcpy(h_out, lcb::g_stage_prof, 12 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return LC_E_CUDA;
  cudaMemset(lcb::g_stage_prof, 0, 16 * sizeof(unsigned long long));
  return LC_OK;
}
