// raas_decode.cuh — the fused RaaS decode-step kernel (sm_100a), warp-specialized.
//
// One launch = one decode step of one layer (handle) for every unit (request, kv-head):
//   a1 slot selection (from the plan computed at the end of the previous step)
//   a2 in-place write of k_new / v_new into the slot (smem tile + HBM store)
//   a3 split-K flash-decode over the resident pages        (consumer warps, mma.sync bf16)
//   a4 page-max logits M_{h,p}                             (consumer warps)
//   a5 LSE combine across splits, bf16 output              (combine warp, last split of a unit)
//   a6 stamp: ts[p] = t iff max_h M_{h,p} - LSE_h > log2(alpha)   (combine warp)
//   a7 next victim = argmin_{unpinned} (ts, start_pos); next plan  (combine warp)
// PAPER.md §3.3 :143-151, App. B :358-398; readings D1-D20 in DESIGN.md.
//
// CTA (persistent, one per SM; tiles (unit, split) of SP pages, static order blockIdx + k*grid):
//   warp 0         producer: per page ONE 1-D bulk async copy (TMA engine) of the page's K and
//                  V rows (2 x 16 x D bf16, contiguous, stored pre-swizzled) into a ring of S
//                  stages, one lane per page; per tile a bulk copy of the unit's q rows;
//                  prefetches the next tile's plan / page counts.
//   warp 1         merge: merges the consumers' per-tile softmax states (smem), publishes the
//                  tile's split-K partial (release/acquire counter per unit) and queues a unit
//                  whose last split it published.
//   warp 2         combine: a5-a7 for each queued unit.  Neither warp consumes ring stages, so
//                  their latency does not stall HBM.
//   warps 3..NC+2  consumers: ring position j goes to consumer j % NC; per page
//                  S^T = K_page Q^T and O^T += V_page^T P^T on mma.sync m16n8k16 (16 tokens = M,
//                  the <= 8 q-heads of the GQA group = N), online softmax in fp32 registers.
//
// Instantiations (template <D, NC, S, TOKD, GEN, CL, FM>, chosen per handle in raas_api.cu):
// lean (the default method, options compiled out); FM = F_QUEST / F_TOPR / F_TSC / F_HYB (one
// option compiled in); GEN (every option decided at run time); TOKD (deferred token level);
// CL (cluster schedule of lean for small batches); NC = 4, S = 8 (half-size CTAs, L <= 256).
#pragma once

#ifndef RAAS_MINB
#define RAAS_MINB 1  // resident CTAs per SM the kernel is compiled for (register budget)
#endif
#ifndef RAAS_PRE
#define RAAS_PRE 0  // pages issued before griddepcontrol.wait (early start); 0: see the producer
#endif
#ifndef RAAS_CL
#define RAAS_CL 1  // compile the cluster schedule (DecodeParams::cl) into the kernels
#endif
#ifndef RAAS_DEP
#define RAAS_DEP 2  // consumer deposit buffers per consumer (see DecodeLayout::NDEP)
#endif
#ifndef RAAS_PREFETCH_TILES
#define RAAS_PREFETCH_TILES 4  // cap on the owned tiles warmed in L2 before griddepcontrol.wait
#endif

namespace raas {

#ifdef RAAS_DBG_TIMING  // tuning experiment: per-CTA cycle accounting of the pipeline waits
__device__ unsigned long long g_raas_dbg[1024][16];
__device__ unsigned long long g_raas_dbg_unit[4096][4];  // cta, pushed, combine start, end
__device__ unsigned long long g_raas_dbg_comb[4096][4];  // combine phases: LSE done, out done, stamps done, end
// multi-launch timeline: [launch slot][cta] = {entry, after griddepcontrol.wait, producer end, exit}
__device__ unsigned long long g_raas_tl[8][256][4];
__device__ __forceinline__ long long dbg_clock() { return clock64(); }
__device__ __forceinline__ void dbg_add(int slot, long long t0) {
  if ((threadIdx.x & 31) == 0) atomicAdd(&g_raas_dbg[blockIdx.x][slot], (unsigned long long)(clock64() - t0));
}
__device__ __forceinline__ unsigned long long dbg_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#else
__device__ __forceinline__ unsigned long long dbg_gtimer() { return 0; }
__device__ __forceinline__ long long dbg_clock() { return 0; }
__device__ __forceinline__ void dbg_add(int, long long) {}
#endif
#ifdef RAAS_DBG_TIMING
#define RAAS_COMB_MARK(i) \
  do { if (lane == 0 && unit < 4096) g_raas_dbg_comb[unit][i] = dbg_gtimer(); } while (0)
__device__ long long g_raas_dbg_cyc[4096][8];  // combine: SM cycles at fine marks
#define RAAS_CYC(i) \
  do { if (lane == 0 && unit < 4096) g_raas_dbg_cyc[unit][i] = clock64(); } while (0)
#else
#define RAAS_CYC(i) do {} while (0)
#define RAAS_COMB_MARK(i) do {} while (0)
#endif
#define RAAS_TIMED(slot, stmt)          \
  do {                                  \
    const long long t0_ = dbg_clock();  \
    stmt;                               \
    dbg_add(slot, t0_);                 \
  } while (0)

// Checked builds (-DRAAS_CHECKED; tests/test_gpu_parity.py::test_checked_build_bounds): device
// bounds checks on every index the step derives from its state, reported in the status word
// (bit 8, plus bit 9 + site).  Release builds compile them out.
#ifdef RAAS_CHECKED
#define RAAS_CHK(cond, site) \
  do { if (!(cond)) atomicOr(p.status, 0x100u | (1u << (9 + (site)))); } while (0)
#else
#define RAAS_CHK(cond, site) do {} while (0)
#endif

constexpr int PUB_ACC_OFF = MAX_GROUP * 8;  // cluster schedule: acc after the (m, l) pairs
constexpr int FLAG_FIRST = 1;  // first page of this tile for the consuming warp
constexpr int FLAG_LAST = 2;   // last page of this tile for the consuming warp
constexpr int FLAG_END = 4;    // no more work
constexpr int FLAG_SKIP = 8;   // padding position (keeps every tile aligned to the NC consumers)
constexpr int CQ_OWNED = 1 << 30;  // combine-queue tag: all splits were processed by this CTA
constexpr int CQ_OUTDONE = 1 << 29;  // tag: the merge warp already wrote out; LSE in the slot
constexpr int CQ_UNIT_BITS = 20;   // entry = unit | nse << 20 | outdone << 29 | owned << 30
constexpr int CQ_NSE_MASK = (1 << 9) - 1;  // nse <= MAX_SPLITS < 512

// The split combine (a5) is a running merge in split order, per head h and element d:
//   m' = max(m, m_s);  f_a = 2^(m - m'), f_b = 2^(m_s - m')  (m' = -inf -> 0 in the exponent)
//   l = l f_a + l_s f_b;  acc = acc f_a + acc_s f_b;  LSE = m + log2 l;  out = acc (1 / l).
// The merge warp folds an owned unit's splits this way as they finish (no partials in HBM/L2),
// the combine warp folds a shared unit's published partials the same way, with the same
// operations, so a unit's result does not depend on which path (i.e. on the schedule) ran it.
__device__ __forceinline__ void merge_factors(float m, float ms, float& mn, float& fa, float& fb) {
  mn = fmaxf(m, ms);
  const float sf = mn == -INFINITY ? 0.f : mn;
  fa = fast_exp2(m - sf);
  fb = fast_exp2(ms - sf);
}

// Tile schedule of one CTA (it never changes numerics: the split arithmetic is schedule-free).
// With G CTAs, CTA b first streams the whole units [b*fu, (b+1)*fu), fu = units / G, whose
// splits are combined inside the CTA; then the split tiles of the R = units - fu*G remaining
// ("shared") units are grabbed dynamically from a global counter, so CTAs that streamed
// faster take more of them and the kernel ends balanced.  The last CTA to exit resets the
// counter for the next launch.
// Cluster schedule (cl): CTA b streams tile b only, i.e. split b % nsplit of unit b / nsplit
// (the cluster of the unit's nsplit consecutive CTAs).
struct TileSched {
  int b, G, fu, nsplit, n_owned, n_shared_tiles, shared_base, i_owned;
  bool cl;
  __device__ TileSched(int units, int nsplit_, int G_, int b_, bool cl_)
      : b(b_), G(G_), nsplit(nsplit_), cl(cl_) {
    fu = cl ? 0 : units / G;
    n_owned = fu * nsplit;
    n_shared_tiles = cl ? 0 : (units - fu * G) * nsplit;
    shared_base = fu * G * nsplit;
    i_owned = 0;
  }
  // next tile for this CTA (warp-uniform), -1 when none is left
  __device__ int next(int* grab, int lane, bool& owned) {
    if (cl) {
      owned = false;
      return i_owned++ == 0 ? b : -1;
    }
    if (i_owned < n_owned) {
      owned = true;
      return b * n_owned + i_owned++;
    }
    // a grabbed tile of a one-split unit is the whole unit: it takes the owned path (out and
    // LSE from the merge warp, no partial through L2), whichever CTA grabs it
    owned = nsplit == 1;
    if (n_shared_tiles == 0) return -1;
    int x = 0;
    if (lane == 0) x = atomicAdd(grab, 1);
    x = __shfl_sync(0xffffffffu, x, 0);
    return x < n_shared_tiles ? shared_base + x : -1;
  }
};

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint32_t bar, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(n) : "memory");
}
// 1-D bulk copy global -> shared (size multiple of 16), completion counted on `bar`.
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// 1-D bulk copy with an L2 eviction-policy hint (KV pages: evict-first, read once per step)
__device__ __forceinline__ void bulk_load_hint(uint32_t dst, const void* src, uint32_t bytes,
                                               uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
// order-preserving float <-> uint32 (0 is below every float: the identity of atomicMax)
__device__ __forceinline__ uint32_t order_f32(float x) {
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unorder_f32(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds_f32x4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

template <int D, int NC, int S, bool TOKD = false, bool QTR = false>
struct DecodeLayout {
  static constexpr int KS = D / 16;
  static constexpr int TILE = PAGE * D * 2;  // one K (or V) page
  // tokd: + the ts/start trailer; QTR (the generic kernel): room for the Quest mode's per-page
  // min / max key rows (2 x D bf16) that follow the page's V rows in HBM
  static constexpr int STAGE = 2 * TILE + (TOKD ? 128 : 0) + (QTR ? 4 * D : 0);
  static constexpr int QBUF = MAX_GROUP * D * 2;
  static constexpr int FRAG = KS * 4 + 4;  // floats per lane in a consumer's deposit
  static constexpr int DEPOSIT = FRAG * 32 * 4;
  static constexpr int OFF_RING = 0;
  static constexpr int OFF_Q = OFF_RING + S * STAGE;
  static constexpr int OFF_MERGE = OFF_Q + 2 * QBUF;
  // consumer deposits: one buffer per consumer (RAAS_DEP 1: a consumer waits until the merge
  // warp has read its previous tile's deposit; the smem goes to ring stages) or one per tile
  // parity (RAAS_DEP 2)
  static constexpr int NDEP = RAAS_DEP;
  static constexpr int OFF_SCR = OFF_MERGE + NDEP * NC * DEPOSIT;         // combine scratch
  static constexpr int SCR = MAX_SPLITS * MAX_GROUP * 8 + 6 * MAX_GROUP * 4;
  static constexpr int OFF_SINFO = OFF_SCR + SCR;                          // int4[2] per stage
  static constexpr int OFF_TINFO = OFF_SINFO + S * 32;                     // int4[3] per parity
  static constexpr int CQ = 16;                                            // combine queue
  static constexpr int OFF_CQ = OFF_TINFO + 2 * 48;  // int[CQ] unit ids, then the pop counter
  // deferred token level (tokd): per stage the tile's 16 ts + 16 start values; per parity the
  // previous step's q and LSE; per (parity, consumer) the tile's victim candidate
  static constexpr int OFF_LSEQ = (OFF_CQ + CQ * 4 + 32 + 15) / 16 * 16;   // float[CQ][MAX_GROUP]
  static constexpr int OFF_TSB = (OFF_LSEQ + CQ * MAX_GROUP * 4 + 127) / 128 * 128;
  static constexpr int OFF_CAND = OFF_TSB;
  static constexpr int OFF_QP = OFF_CAND + (TOKD ? 2 * NC * 16 : 0);
  static constexpr int QPBUF = QBUF + 32;  // q_prev rows, then 8 floats of LSE
  static constexpr int OFF_BAR = (OFF_QP + (TOKD ? 2 * QPBUF : 0) + 127) / 128 * 128;
  // After its END sentinel (the NC sentinels take NC consecutive ring positions, hence distinct
  // stages) no stage is written again, so for D = 128 a consumer joins the combine pool with
  // its sentinel's stage as scratch (the kernel's tail is the combines of the last units: more
  // poppers, shorter tail).
  static constexpr bool JOIN = STAGE >= SCR && S >= NC;
  static constexpr int NPOP = 1 + (JOIN ? NC : 0);
  static_assert(CQ >= NPOP, "a popper may wait at most one queue phase ahead");
  // full[S], empty[S], qfull[2], mfull[2], tfree[2], cq_full[CQ], cq_empty[CQ], clfull
  static constexpr int NBAR = 2 * S + 6 + 2 * CQ + 1;
  // cluster schedule (p.cl): the tile's split partial, published in this CTA's merge area once
  // the merge warp has read the (only) tile's deposits: float2 (m, l)[MAX_GROUP], then
  // float acc[g][D]; read by the cluster's leader through distributed shared memory
  // cluster schedule (p.cl): the leader receives split s's partial at OFF_RECV + s * RECV_SLOT,
  // the second half of the deposit area (each CTA streams one tile: only deposit parity 0 is used)
  static constexpr int RECV_SLOT = PUB_ACC_OFF + MAX_GROUP * D * 4;
  static constexpr int OFF_RECV = OFF_MERGE + NC * DEPOSIT;
  static constexpr bool CL_OK = NDEP == 2 && 8 * RECV_SLOT <= NC * DEPOSIT;
  static constexpr int BYTES = OFF_BAR + NBAR * 8;
  static constexpr int SMEM = BYTES + 1024;  // + alignment slack
  static constexpr int THREADS = (NC + 3) * 32;  // producer, merge, combine, NC consumers
};

// ---------------------------------------------------------------------------------------------
// a5-a7 for one unit, by one warp, after all its splits have published their partials.
// ---------------------------------------------------------------------------------------------
// Feature masks of the specialised instantiations (one option beside the default method each;
// GEN decides every option at run time): Quest scores, top-r rule, per-request tables, hybrid
constexpr int F_QUEST = 1, F_TOPR = 2, F_TSC = 4, F_HYB = 8;

template <int D, bool GEN, int FM = 0>
__device__ __forceinline__ void combine_unit(const DecodeParams& p, int unit, int nse, uint32_t scr,
                                             int lane, bool outdone, bool CL = false, uint32_t pub = 0,
                                             uint32_t clbar = 0) {
  // CL (cluster schedule): the cluster's CTA s stored split s's partial into this (leader) CTA's
  // receive area `pub` (slot s, distributed shared memory stores) before arriving on `clbar`
  // (release / acquire at cluster scope); the arithmetic below is the same as for partials
  // read from L2, so results do not depend on the schedule
  constexpr int RSLOT = PUB_ACC_OFF + MAX_GROUP * D * 4;
  if (CL) mbar_wait_cluster(clbar, 0);
  // outdone: the merge warp already folded the splits and wrote out; the LSE is in scr_lse
  // GEN = false: the default method (page = 16, alpha rule, one table per kv-head) with the
  // optional rules compiled out; GEN = true: every option decided at run time
  const bool tscope = (GEN || (FM & F_TSC)) && p.table_scope != 0;
  const bool topr = (GEN || (FM & F_TOPR)) && p.stamp_rule == 1;
  // Latency-oriented: the plan, the split statistics, the first block of split partials and
  // the first 128 pages' metadata are all requested before any of them is used (nse comes with
  // the queue entry), so a unit costs ~one dependent L2 round trip before its stores.
  const int C = p.Ce, g = p.g;  // metadata entries: pages, or token slots (ep = 1)
  const int NE = nse * g;
  const uint32_t scr_w = scr;                                   // float[nse][g] split weights
  const uint32_t scr_lse = scr + MAX_SPLITS * MAX_GROUP * 8;    // float[g]
  const uint32_t scr_inv = scr_lse + MAX_GROUP * 4;             // float[g]
  const float2* ml_g = p.part_ml + (size_t)unit * p.nsplit * g;
#ifdef RAAS_DBG_NOCOMB  // upper-bound experiment: an owned unit's combine costs ~nothing (FIFO state)
  if (outdone) {
    if (lane == 0) {
      const int4 pl0 = __ldcg(p.plan + unit);
      const int np0 = __ldg(p.npin + unit), Cc = p.C;
      const int vic = np0 + ((pl0.x - np0 + 1) % (Cc - np0));
      p.cnt[(size_t)unit * Cc + pl0.x] = (pl0.y & 0xffff) + 1;
      p.plan[unit] = next_plan(pl0.x, (pl0.y & 0xffff) + 1, pl0.z, Cc, pl0.w, vic, p.status, PAGE);
    }
    return;
  }
#endif
#ifdef RAAS_DBG_COMBDELAY  // sensitivity probe: a longer owned-unit (or, _SH, shared-unit) combine
#ifdef RAAS_DBG_COMBDELAY_SH
  if (!outdone) {
#else
  if (outdone) {
#endif
    const long long t0 = clock64();
    while (clock64() - t0 < RAAS_DBG_COMBDELAY) {
    }
  }
#endif
  RAAS_CYC(0);
  RAAS_CYC(1);
  const int4 pl = __ldcg(p.plan + unit);
  const int npin = __ldg(p.npin + unit);
  float2 mla[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = 32 * k + lane;
    mla[k] = (outdone || i >= NE) ? make_float2(-INFINITY, 0.f)
             : CL ? make_float2(lds_f32(pub + (i / g) * RSLOT + 8 * (i % g)),
                                lds_f32(pub + (i / g) * RSLOT + 8 * (i % g) + 4))
                  : __ldcg(ml_g + i);
  }
  // page metadata for a6/a7 (bounded by C, masked by the plan's page count later)
  constexpr int PPL = 4;  // pages per lane per chunk
  int tsv[PPL], stv[PPL];
  float pmv[PPL][MAX_GROUP];
  // table_scope 1 (D25): once every kv-head of the request has combined, the last one decides
  // for all of them from the request-wide page scores req_x (then pmv[i][0], with LSE 0)
  const int req = unit / p.n_kv;
  uint32_t* const rx = p.req_x + (size_t)req * C;
  bool rq = false;
  auto load_meta = [&](int pc, int lim) {
#pragma unroll
    for (int i = 0; i < PPL; ++i) {
      const int pg = pc + 32 * i + lane;
      const bool ok = pg < lim;
      const size_t ix = (size_t)unit * C + pg;
      tsv[i] = ok ? __ldcg(p.ts + ix) : 0;
      stv[i] = ok ? __ldcg(p.start + ix) : 0;
      if (rq) {
        pmv[i][0] = (ok && pg >= npin) ? unorder_f32(__ldcg(rx + pg)) : -INFINITY;
#pragma unroll
        for (int h = 1; h < MAX_GROUP; ++h) pmv[i][h] = -INFINITY;
      } else {
#pragma unroll
        for (int h = 0; h < MAX_GROUP; ++h)
          pmv[i][h] = (ok && h < g) ? __ldcg(p.pmax + ix * g + h) : -INFINITY;
      }
    }
  };
  load_meta(0, C);
  RAAS_CYC(2);
  // first block of split partials: 4 float4 chunks per lane x 2 splits
  constexpr int CPH = D / 4;                   // chunks per head
  constexpr int CB = 4, SG = 2;
  const int nch = g * CPH;
  const float* acc_g = p.part_acc + (size_t)unit * p.nsplit * g * D;
  float4 v[CB][SG];
  auto load_acc = [&](int cb, int s0) {
#pragma unroll
    for (int i = 0; i < CB; ++i) {
      const int c = lane + 32 * (cb + i), h = c / CPH, d4 = c - h * CPH;
#pragma unroll
      for (int u = 0; u < SG; ++u) {
        const bool ok = !outdone && c < nch && s0 + u < nse;
        v[i][u] = !ok ? make_float4(0.f, 0.f, 0.f, 0.f)
                  : CL ? lds_f32x4(pub + (s0 + u) * RSLOT + PUB_ACC_OFF + (h * D + 4 * d4) * 4)
                       : __ldcg(reinterpret_cast<const float4*>(acc_g + ((size_t)(s0 + u) * g + h) * D) + d4);
      }
    }
  };
  load_acc(0, 0);
  RAAS_CYC(3);
  // ---- a5 (1): running merge of the split statistics -> per-split factors, LSE, 1 / l ----
  if (!outdone) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int i = 32 * k + lane;
      if (i < NE) { sts_f32(scr_w + 8 * i, mla[k].x); sts_f32(scr_w + 8 * i + 4, mla[k].y); }
    }
    for (int i = 64 + lane; i < NE; i += 32) {  // more than 64 (split, head) pairs
      const float2 ml = CL ? make_float2(lds_f32(pub + (i / g) * RSLOT + 8 * (i % g)),
                                         lds_f32(pub + (i / g) * RSLOT + 8 * (i % g) + 4))
                           : __ldcg(ml_g + i);
      sts_f32(scr_w + 8 * i, ml.x);
      sts_f32(scr_w + 8 * i + 4, ml.y);
    }
  }
  const int slot = pl.x, off = pl.y & 0xffff, evicting = pl.y >> 16;
  const int used_eff = pl.z, t = pl.w;
  RAAS_CHK(unit >= 0 && unit < p.units && nse >= 1 && nse <= p.nsplit && slot >= 0 && slot < C &&
               off >= 0 && off < (GEN ? p.ep : PAGE) && used_eff > slot && used_eff <= C &&
               npin >= 0 && npin <= used_eff, 3);
  __syncwarp();
  if (!outdone && lane < g) {  // (m_s, l_s) of split s are replaced by its factors (f_a, f_b)
    float m = -INFINITY, l = 0.f;
    for (int s = 0; s < nse; ++s) {
      const uint32_t a = scr_w + 8 * (s * g + lane);
      float mn, fa, fb;
      merge_factors(m, lds_f32(a), mn, fa, fb);
      l = fmaf(l, fa, __fmul_rn(lds_f32(a + 4), fb));
      m = mn;
      sts_f32(a, fa);
      sts_f32(a + 4, fb);
    }
    sts_f32(scr_lse + 4 * lane, m + log2f(l));
    sts_f32(scr_inv + 4 * lane, 1.f / l);
  }
  __syncwarp();
  RAAS_COMB_MARK(0);
  RAAS_CYC(4);
  float lse[MAX_GROUP];
#pragma unroll
  for (int h = 0; h < MAX_GROUP; ++h) lse[h] = h < g ? lds_f32(scr_lse + 4 * h) : 0.f;
  // page score x_p = max_h (score_hp - LSE_h) (log2 domain).  Rule 0: stamp iff x_p > log2 a
  // (strict, D3).  Rule 1 (top-r, PAPER.md :135, reading D23): stamp the k = ceil(r n) pages with
  // the largest (x_p, -start_pos) among the n unpinned resident pages.
  auto page_x = [&](int i) {
    float x = -INFINITY;
#pragma unroll
    for (int h = 0; h < MAX_GROUP; ++h)
      if (h < g) x = fmaxf(x, pmv[i][h] - lse[h]);
    return x;
  };
  if (tscope) {
    // table_scope 1 (D25): fold this kv-head's page scores into the request-wide maximum
    // early, so the reductions drain while the output is combined
    for (int pc = 0; pc < used_eff; pc += 32 * PPL) {
      if (pc > 0) load_meta(pc, used_eff);
#pragma unroll
      for (int i = 0; i < PPL; ++i) {
        const int pg = pc + 32 * i + lane;
        if (pg >= npin && pg < used_eff) atomicMax(rx + pg, order_f32(page_x(i)));
      }
    }
    // ... then counts itself in; the last one decides for the request (its loads of req_x
    // overlap the output combine).  The release of lane 0's counter increment covers the
    // other lanes' reductions, ordered before it by __syncwarp.
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      last = atom_add_acq_rel_gpu(p.req_ctr + req, 1) == p.n_kv - 1;
      p.counter[unit] = 0;
      if (evicting) atomicAdd(p.stats + 2, 1ull);
      atomicAdd(p.stats + 3, 1ull);
      if (last) p.req_ctr[req] = 0;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    __syncwarp();  // orders lane 0's acquire before the other lanes' loads of req_x
    if (last) {
      rq = true;
      load_meta(0, used_eff);
    }
  }
  // ---- a5 (2): out[h][d] = acc[h][d] / l_h, acc folded in split order ----
  for (int cb = 0; !outdone && 32 * cb < nch; cb += CB) {
    float4 o[CB];
#pragma unroll
    for (int i = 0; i < CB; ++i) o[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < nse; s0 += SG) {
      if (cb > 0 || s0 > 0) load_acc(cb, s0);
#pragma unroll
      for (int i = 0; i < CB; ++i) {
        const int c = lane + 32 * (cb + i), h = c / CPH;
        if (c < nch) {
#pragma unroll
          for (int u = 0; u < SG; ++u) {
            if (s0 + u < nse) {
              const uint32_t fa_a = scr_w + 8 * ((s0 + u) * g + h);
              const float fa = lds_f32(fa_a), fb = lds_f32(fa_a + 4);
              o[i].x = fmaf(o[i].x, fa, __fmul_rn(v[i][u].x, fb));
              o[i].y = fmaf(o[i].y, fa, __fmul_rn(v[i][u].y, fb));
              o[i].z = fmaf(o[i].z, fa, __fmul_rn(v[i][u].z, fb));
              o[i].w = fmaf(o[i].w, fa, __fmul_rn(v[i][u].w, fb));
            }
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CB; ++i) {
      const int c = lane + 32 * (cb + i), h = c / CPH, d4 = c - h * CPH;
      if (c < nch) {
        const float inv = lds_f32(scr_inv + 4 * h);
        const uint2 pk = make_uint2(pack_bf16x2(o[i].x * inv, o[i].y * inv),
                                    pack_bf16x2(o[i].z * inv, o[i].w * inv));
        *reinterpret_cast<uint2*>(p.out + (size_t)(unit * g + h) * D + 4 * d4) = pk;
      }
    }
  }
  // ---- a6: stamp; a2 metadata of the write slot; a7 candidates ----
  RAAS_COMB_MARK(1);
  if (tscope && !rq) return;  // another kv-head of the request decides
  if (rq) {
#pragma unroll
    for (int h = 0; h < MAX_GROUP; ++h) lse[h] = 0.f;  // req_x already holds normalised scores
  }
  const int nrep = tscope ? p.n_kv : 1;   // metadata replicas this warp writes
  const int unit0 = tscope ? req * p.n_kv : unit;
  auto page_key = [&](float x, int st) {  // larger key = ranked first; valid keys are > 0
    const uint32_t b = __float_as_uint(x);
    const uint32_t sx = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return (static_cast<unsigned long long>(sx) << 32) | (0xffffffffu - static_cast<uint32_t>(st));
  };
  unsigned long long kth = 0;
  if (topr) {
    // pass 1: keys of the decision pages -> scratch (the split weights are no longer needed)
    const uint32_t scr_key = scr, scr_hist = scr + 8 * 512;
    int nd = 0;
    for (int pc = 0; pc < used_eff; pc += 32 * PPL) {
      if (pc > 0) load_meta(pc, used_eff);
#pragma unroll
      for (int i = 0; i < PPL; ++i) {
        const int pg = pc + 32 * i + lane;
        if (pg < used_eff) {
          const int st_p = (pg == slot && off == 0) ? t : stv[i];
          const unsigned long long key = pg >= npin ? page_key(page_x(i), st_p) : 0ull;
          nd += pg >= npin ? 1 : 0;
          asm volatile("st.shared.u64 [%0], %1;" ::"r"(scr_key + 8 * pg), "l"(key) : "memory");
        }
      }
    }
    nd = warp_sum_i(nd);
    int krem = (int)ceilf(p.top_r * (float)nd);  // fp32, as the oracle (D23)
    krem = krem < 0 ? 0 : (krem > nd ? nd : krem);
    __syncwarp();
    if (krem > 0) {
      // keys are unique (start positions differ): exactly k keys are >= kth
      kth = warp_kth_largest(scr_key, scr_hist, used_eff, krem, lane);

    } else {
      kth = ~0ull;  // nothing stamped
    }
    if (used_eff > 32 * PPL) load_meta(0, used_eff);
  }
  Cand best{~0ull, -1};
  int n_stamp = 0, n_dec = 0;
  for (int pc = 0; pc < used_eff; pc += 32 * PPL) {
    if (pc > 0) load_meta(pc, used_eff);
#pragma unroll
    for (int i = 0; i < PPL; ++i) {
      const int pg = pc + 32 * i + lane;
      if (pg < used_eff) {
        int ts_p = tsv[i], st_p = stv[i];
        const bool is_slot = pg == slot;
        if (is_slot) {
          if (off == 0) st_p = t;
          for (int r = 0; r < nrep; ++r) {
            const size_t ix = (size_t)(unit0 + r) * C + pg;
            if (off == 0) p.start[ix] = t;
            p.cnt[ix] = off + 1;
          }
        }
        if (pg >= npin) {
          const float x = page_x(i);
          const bool stamp = topr ? page_key(x, st_p) >= kth
                                               : x > p.log2_alpha;  // strict (D3)
          ++n_dec;
          n_stamp += stamp ? 1 : 0;
          if (stamp || is_slot) {  // stamp, or write refresh (D8)
            ts_p = t;
            for (int r = 0; r < nrep; ++r) p.ts[(size_t)(unit0 + r) * C + pg] = t;
          }
          if (rq) rx[pg] = 0u;  // reset for the next step
          cand_update(best, cand_key(ts_p, st_p), pg);
        }
      }
    }
  }
  RAAS_COMB_MARK(2);
  RAAS_CYC(5);
  const int victim = warp_argmin_page(best);
  RAAS_CHK(victim >= -1 && victim < C && (victim < 0 || victim >= npin), 4);
  n_stamp = warp_sum_i(n_stamp);
  n_dec = warp_sum_i(n_dec);
  RAAS_COMB_MARK(3);
  if (lane == 0) {
    const int4 np = next_plan(slot, off + 1, used_eff, C, t, victim, p.status, GEN ? p.ep : PAGE);
    for (int r = 0; r < nrep; ++r) p.plan[unit0 + r] = np;
    atomicAdd(p.stats + 0, (unsigned long long)n_stamp);
    atomicAdd(p.stats + 1, (unsigned long long)n_dec);
    if (!rq) {
      p.counter[unit] = 0;
      if (evicting) atomicAdd(p.stats + 2, 1ull);
      atomicAdd(p.stats + 3, 1ull);
    }
  }
  RAAS_CYC(6);
}


// ---------------------------------------------------------------------------------------------
// Cluster schedule (small batches, the default method): a5-a7 for the cluster's unit by the
// leader's combine warp with no L2 round trip on its critical path.  The unit's plan, pinned
// count and per-page (ts, start) were loaded at kernel start (`cm`: they are the previous step's
// state); the splits' (m, l, acc) partials and the page maxima arrive in this CTA's shared
// memory from the cluster's merge warps / consumers (`recv`, `pmx`).  Every operation and its
// order are those of combine_unit (split-order running merge, strict threshold, (ts, start)
// argmin), so results are bitwise those of the default schedule.
// ---------------------------------------------------------------------------------------------
constexpr int CLM = 8;  // pages per lane the preloaded metadata covers (C <= 256)
struct ClMeta {
  int4 pl;
  int npin;
  int ts[CLM], st[CLM];
};
template <int D>
__device__ __forceinline__ void combine_unit_cl(const DecodeParams& p, int unit, int nse, uint32_t scr,
                                                int lane, uint32_t recv, uint32_t pmx,
                                                uint32_t clbar, const ClMeta& cm) {
  constexpr int RSLOT = PUB_ACC_OFF + MAX_GROUP * D * 4;
  const int C = p.C, g = p.g;
  const uint32_t scr_w = scr;                                   // float2[nse][g] split factors
  const uint32_t scr_lse = scr + MAX_SPLITS * MAX_GROUP * 8;    // float[g]
  const uint32_t scr_inv = scr_lse + MAX_GROUP * 4;             // float[g]
  mbar_wait_cluster(clbar, 0);  // every split's partial and page maxima are here
  RAAS_COMB_MARK(0);
  // ---- a5 (1): running merge of the split statistics -> factors, LSE, 1 / l ----
  if (lane < g) {
    float m = -INFINITY, l = 0.f;
    for (int s = 0; s < nse; ++s) {
      const uint32_t a = recv + s * RSLOT + 8 * lane;
      float mn, fa, fb;
      merge_factors(m, lds_f32(a), mn, fa, fb);
      l = fmaf(l, fa, __fmul_rn(lds_f32(a + 4), fb));
      m = mn;
      sts_f32(scr_w + 8 * (s * g + lane), fa);
      sts_f32(scr_w + 8 * (s * g + lane) + 4, fb);
    }
    sts_f32(scr_lse + 4 * lane, m + log2f(l));
    sts_f32(scr_inv + 4 * lane, 1.f / l);
  }
  __syncwarp();
  // ---- a5 (2): out[h][d] = acc[h][d] / l_h, acc folded in split order ----
  constexpr int CPH = D / 4;  // float4 chunks per head; a lane's 4 chunks per round share a head
  const int nch = g * CPH;
  for (int c0 = 4 * lane; c0 < nch; c0 += 128) {  // 4 consecutive chunks per lane per round
    const int h = c0 / CPH, d40 = c0 - h * CPH;
    float4 o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < nse; ++s) {
      const float fa = lds_f32(scr_w + 8 * (s * g + h)), fb = lds_f32(scr_w + 8 * (s * g + h) + 4);
      float4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = lds_f32x4(recv + s * RSLOT + PUB_ACC_OFF + (h * D + 4 * (d40 + k)) * 4);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        o[k].x = fmaf(o[k].x, fa, __fmul_rn(v[k].x, fb));
        o[k].y = fmaf(o[k].y, fa, __fmul_rn(v[k].y, fb));
        o[k].z = fmaf(o[k].z, fa, __fmul_rn(v[k].z, fb));
        o[k].w = fmaf(o[k].w, fa, __fmul_rn(v[k].w, fb));
      }
    }
    const float inv = lds_f32(scr_inv + 4 * h);
#pragma unroll
    for (int k = 0; k < 4; k += 2)
      *reinterpret_cast<uint4*>(p.out + (size_t)(unit * g + h) * D + 4 * (d40 + k)) =
          make_uint4(pack_bf16x2(o[k].x * inv, o[k].y * inv), pack_bf16x2(o[k].z * inv, o[k].w * inv),
                     pack_bf16x2(o[k + 1].x * inv, o[k + 1].y * inv),
                     pack_bf16x2(o[k + 1].z * inv, o[k + 1].w * inv));
  }
  // ---- a6: stamp; a2 metadata of the write slot; a7 candidates ----
  RAAS_COMB_MARK(1);
  float lse[MAX_GROUP];
#pragma unroll
  for (int h = 0; h < MAX_GROUP; ++h) lse[h] = h < g ? lds_f32(scr_lse + 4 * h) : 0.f;
  const int4 pl = cm.pl;
  const int slot = pl.x, off = pl.y & 0xffff, evicting = pl.y >> 16;
  const int used_eff = pl.z, t = pl.w, npin = cm.npin;
  Cand best{~0ull, -1};
  int n_stamp = 0, n_dec = 0;
#pragma unroll
  for (int i = 0; i < CLM; ++i) {
    const int pg = 32 * i + lane;
    if (pg < used_eff) {
      int ts_p = cm.ts[i], st_p = cm.st[i];
      const bool is_slot = pg == slot;
      const size_t ix = (size_t)unit * C + pg;
      if (is_slot) {
        if (off == 0) {
          st_p = t;
          p.start[ix] = t;
        }
        p.cnt[ix] = off + 1;
      }
      if (pg >= npin) {
        float x = -INFINITY;
#pragma unroll
        for (int h = 0; h < MAX_GROUP; ++h)
          if (h < g) x = fmaxf(x, lds_f32(pmx + 4 * (pg * g + h)) - lse[h]);
        const bool stamp = x > p.log2_alpha;  // strict (D3)
        ++n_dec;
        n_stamp += stamp ? 1 : 0;
        if (stamp || is_slot) {  // stamp, or write refresh (D8)
          ts_p = t;
          p.ts[ix] = t;
        }
        cand_update(best, cand_key(ts_p, st_p), pg);
      }
    }
  }
  RAAS_COMB_MARK(2);
  const int victim = warp_argmin_page(best);
  n_stamp = warp_sum_i(n_stamp);
  n_dec = warp_sum_i(n_dec);
  RAAS_COMB_MARK(3);
  if (lane == 0) {
    p.plan[unit] = next_plan(slot, off + 1, used_eff, C, t, victim, p.status, PAGE);
    atomicAdd(p.stats + 0, (unsigned long long)n_stamp);
    atomicAdd(p.stats + 1, (unsigned long long)n_dec);
    p.counter[unit] = 0;
    if (evicting) atomicAdd(p.stats + 2, 1ull);
    atomicAdd(p.stats + 3, 1ull);
  }
}

// ---------------------------------------------------------------------------------------------
// Deferred token-level combine (tokd; NEXT-3): the pass attended the resident rows [0, used)
// and took step t-1's stamp decisions.  Here: victim = min over the splits' candidates (if the
// cache is full), out = softmax over (resident - victim + new token), LSE_t and q_t stored for
// the next pass's decisions, the new token written into its slot.  PAPER.md §3.2 :98-100.
// ---------------------------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ void combine_unit_tok(const DecodeParams& p, int unit, int nse,
                                                 uint32_t scr, int lane) {
  const int C = p.Ce, g = p.g;
  const int NE = nse * g;
  const uint32_t scr_w = scr;                                   // float2[nse][g] (m, l) -> w
  const uint32_t scr_h = scr + MAX_SPLITS * MAX_GROUP * 8;      // per head: M, L, wv, f, wn, inv
  auto hs = [&](int k, int h) { return scr_h + 4 * (k * MAX_GROUP + h); };
  const float2* ml_g = p.part_ml + (size_t)unit * p.nsplit * g;
  const int4 pl = __ldcg(p.plan + unit);  // {fill slot or -1, pending, used rows, t}
  const int used = pl.z, t = pl.w;
  const bool evict = used >= C;
  // split statistics and victim candidates
  for (int i = lane; i < NE; i += 32) {
    const float2 ml = __ldcg(ml_g + i);
    sts_f32(scr_w + 8 * i, ml.x);
    sts_f32(scr_w + 8 * i + 4, ml.y);
  }
  unsigned long long best = ~0ull;
  int vslot = -1;
  for (int i = lane; i < nse; i += 32) {
    const int4 c = __ldcg(p.part_key + (size_t)unit * p.nsplit + i);
    const unsigned long long key = (static_cast<unsigned long long>(static_cast<uint32_t>(c.y)) << 32) |
                                   static_cast<uint32_t>(c.x);
    if (key < best) { best = key; vslot = c.z; }
  }
  {
    const unsigned long long m = warp_min_u64(best);
    const unsigned hit = __ballot_sync(0xffffffffu, best == m);
    vslot = __shfl_sync(0xffffffffu, vslot, __ffs(hit) - 1);
    if (m == ~0ull) vslot = -1;
  }
  int slot = used;
  if (evict) {
    slot = vslot;
    if (slot < 0) {  // no unpinned resident row (cannot happen when P < L)
      if (lane == 0) atomicOr(p.status, 1u);
      slot = C - 1;
    }
  }
  // this lane's channels: q (all heads), the new K row, the victim's K row (swizzled store)
  constexpr int CPL = D / 32;                 // channels per lane
  const int c0 = lane * CPL;
  const int tile = slot >> 4, row = slot & (PAGE - 1);
  __nv_bfloat16* const pg0 = p.kvstore + (size_t)(unit * p.C + tile) * p.pstr;
  const __nv_bfloat16* krow = pg0 + row * D;
  const __nv_bfloat16* vrow = krow + PAGE * D;
  auto swz = [&](int c) { return (((c >> 3) ^ (row & 7)) << 3) | (c & 7); };
  float kn[CPL], kv[CPL];
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    kn[i] = __bfloat162float(p.k_new[(size_t)unit * D + c0 + i]);
    kv[i] = evict ? __bfloat162float(krow[swz(c0 + i)]) : 0.f;
  }
  float sn[MAX_GROUP], sv[MAX_GROUP];
#pragma unroll
  for (int h = 0; h < MAX_GROUP; ++h) {
    float a = 0.f, b = 0.f;
    if (h < g) {
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        const float qv = __bfloat162float(p.q[((size_t)unit * g + h) * D + c0 + i]);
        a += qv * kn[i];
        b += qv * kv[i];
      }
    }
    sn[h] = warp_sum(a) * p.scale_log2;
    sv[h] = warp_sum(b) * p.scale_log2;
  }
  __syncwarp();
  if (lane < g) {  // LSE over the splits (reference 0 when no row was resident)
    float M = -INFINITY;
    for (int s = 0; s < nse; ++s) M = fmaxf(M, lds_f32(scr_w + 8 * (s * g + lane)));
    const float Mr = M == -INFINITY ? 0.f : M;
    float L = 0.f;
    for (int s = 0; s < nse; ++s) {
      const uint32_t a = scr_w + 8 * (s * g + lane);
      const float w = fast_exp2(lds_f32(a) - Mr);
      L += w * lds_f32(a + 4);
      sts_f32(a, w);
    }
    float s_n = sn[0], s_v = sv[0];
#pragma unroll
    for (int h = 1; h < MAX_GROUP; ++h)
      if (h == lane) { s_n = sn[h]; s_v = sv[h]; }
    // minus the victim's row, plus the new token (D9: evict -> write -> attend)
    const float wv = evict ? fast_exp2(s_v - Mr) : 0.f;
    const float M2 = fmaxf(M, s_n);
    const float f = M == -INFINITY ? 0.f : fast_exp2(Mr - M2);
    const float wn = fast_exp2(s_n - M2);
    const float L2 = fmaxf(L - wv, 0.f) * f + wn;
    sts_f32(hs(2, lane), wv);
    sts_f32(hs(3, lane), f);
    sts_f32(hs(4, lane), wn);
    sts_f32(hs(5, lane), 1.f / L2);
    p.lse_prev[(size_t)unit * 8 + lane] = M2 + log2f(L2);  // LSE_t, for the next pass
  }
  __syncwarp();
  // out[h][d] = ((sum_s w_s acc_s - wv v_victim) f + wn v_new) / L'
  constexpr int CPH = D / 4;
  const int nch = g * CPH;
  const float* acc_g = p.part_acc + (size_t)unit * p.nsplit * g * D;
  for (int c = lane; c < nch; c += 32) {
    const int h = c / CPH, d4 = c - h * CPH;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s2 = 0; s2 < nse; ++s2) {
      const float w = lds_f32(scr_w + 8 * (s2 * g + h));
      const float4 a = __ldcg(reinterpret_cast<const float4*>(acc_g + ((size_t)s2 * g + h) * D) + d4);
      o.x += w * a.x; o.y += w * a.y; o.z += w * a.z; o.w += w * a.w;
    }
    const float wv = lds_f32(hs(2, h)), f = lds_f32(hs(3, h)), wn = lds_f32(hs(4, h));
    const float inv = lds_f32(hs(5, h));
    float vv[4], vn[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      vv[i] = evict ? __bfloat162float(vrow[swz(4 * d4 + i)]) : 0.f;
      vn[i] = __bfloat162float(p.v_new[(size_t)unit * D + 4 * d4 + i]);
    }
    o.x = ((o.x - wv * vv[0]) * f + wn * vn[0]) * inv;
    o.y = ((o.y - wv * vv[1]) * f + wn * vn[1]) * inv;
    o.z = ((o.z - wv * vv[2]) * f + wn * vn[2]) * inv;
    o.w = ((o.w - wv * vv[3]) * f + wn * vn[3]) * inv;
    *reinterpret_cast<uint2*>(p.out + (size_t)(unit * g + h) * D + 4 * d4) =
        make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
  }
  // q_t for the next pass's decisions
  {
    const uint4* qs = reinterpret_cast<const uint4*>(p.q + (size_t)unit * g * D);
    uint4* qd = reinterpret_cast<uint4*>(p.q_prev + (size_t)unit * g * D);
    for (int i = lane; i < g * D / 8; i += 32) qd[i] = __ldg(qs + i);
  }
  __syncwarp();  // every lane's reads of the victim's rows are done
  // a2: the new token's K / V into the slot (pre-swizzled rows)
  constexpr int NCH = D / 8;
  if (lane < 2 * NCH) {
    const bool isv = lane >= NCH;
    const int ch = isv ? lane - NCH : lane;
    const uint4 val = __ldg(reinterpret_cast<const uint4*>((isv ? p.v_new : p.k_new) + (size_t)unit * D) + ch);
    *reinterpret_cast<uint4*>(const_cast<__nv_bfloat16*>(isv ? vrow : krow) + ((ch ^ (row & 7)) << 3)) = val;
  }
  if (lane == 0) {
    const size_t ix = (size_t)unit * C + slot;
    p.ts[ix] = t;      // write refresh (D8)
    p.start[ix] = t;   // the token's position
    p.cnt[ix] = 1;
    int32_t* trailer = reinterpret_cast<int32_t*>(pg0 + 2 * PAGE * D);
    trailer[row] = t;
    trailer[PAGE + row] = t;
    const int used2 = evict ? used : used + 1;
    p.plan[unit] = make_int4(used2 < C ? used2 : -1, 1, used2, t + 1);
    p.counter[unit] = 0;
    if (evict) atomicAdd(p.stats + 2, 1ull);
    atomicAdd(p.stats + 3, 1ull);
  }
}

#ifdef RAAS_DBG_TOKD_GLOBAL
__device__ int g_tokd_dbg[16];
#endif
template <int D, int NC, int S, bool TOKD, bool GEN, bool CL = false, int FM = 0>
__global__ void __launch_bounds__(DecodeLayout<D, NC, S, TOKD, GEN || (FM & F_QUEST)>::THREADS,
                                  (NC <= 4 ? 2 : RAAS_MINB))
    raas_decode_kernel(const __grid_constant__ DecodeParams p) {
  // CL: the cluster-schedule instantiation of the default method (small batches); the other
  // instantiations carry none of its code (registers: see DESIGN.md §6)
  // GEN = false (and !TOKD): the default method only (page = 16, exact page score, alpha rule,
  // per-kv-head tables, no Quest-on-prefill); the options' run-time branches are compiled out
  // FM: a specialised instantiation with one option compiled in (F_QUEST: Quest scores, F_TOPR:
  // top-r rule, F_TSC: per-request tables, F_HYB: Quest-on-prefill hybrid), the rest default
  const int quest_k = (GEN || (FM & F_HYB)) ? p.quest_k : 0;
  const int score_mode = GEN ? p.score_mode : ((FM & F_QUEST) ? 1 : 0);
  // TOKD: the deferred token-level instantiation (p.tokd == 1); the page kernel carries none
  // of its code
  static_assert(D == 64 || D == 128, "head_dim");
  using Lay = DecodeLayout<D, NC, S, TOKD, GEN || (FM & F_QUEST)>;
  constexpr int KS = Lay::KS, TILE = Lay::TILE, STAGE = Lay::STAGE;
  constexpr int ROW = 2 * D;  // bytes per token row

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // 128B-swizzle atoms need 1024B alignment
  const uint32_t ring = base + Lay::OFF_RING, qbuf = base + Lay::OFF_Q;
  const uint32_t merge = base + Lay::OFF_MERGE, scr = base + Lay::OFF_SCR;
  const uint32_t lseq = base + Lay::OFF_LSEQ;
  const uint32_t qpb = base + Lay::OFF_QP, cand = base + Lay::OFF_CAND;
  int4* sinfo = reinterpret_cast<int4*>(smem_raw + (base - raw) + Lay::OFF_SINFO);
  int4* tinfo = reinterpret_cast<int4*>(smem_raw + (base - raw) + Lay::OFF_TINFO);
  volatile int* cq = reinterpret_cast<volatile int*>(smem_raw + (base - raw) + Lay::OFF_CQ);
  constexpr int CQ = Lay::CQ;
  int* pop_ctr = reinterpret_cast<int*>(smem_raw + (base - raw) + Lay::OFF_CQ + CQ * 4);
  const uint32_t bar = base + Lay::OFF_BAR;
  auto full = [&](int s) { return bar + 8 * s; };
  auto empty = [&](int s) { return bar + 8 * (S + s); };
  auto qfull = [&](int par) { return bar + 8 * (2 * S + par); };
  auto mfull = [&](int par) { return bar + 8 * (2 * S + 2 + par); };
  auto tfree = [&](int par) { return bar + 8 * (2 * S + 4 + par); };
  auto cqfull = [&](int q) { return bar + 8 * (2 * S + 6 + q); };
  auto cqempty = [&](int q) { return bar + 8 * (2 * S + 6 + CQ + q); };
  const uint32_t clfull = bar + 8 * (2 * S + 6 + 2 * CQ);  // cluster schedule: partials published
  const bool cl = RAAS_CL && Lay::CL_OK && CL && !TOKD && p.cl != 0;
  const uint32_t recv = base + Lay::OFF_RECV;  // cluster schedule: the splits' partials (leader)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef RAAS_DBG_TIMING
  if (threadIdx.x == 0 && blockIdx.x < 256) g_raas_tl[p.dbg_slot & 7][blockIdx.x][0] = dbg_gtimer();
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 32);  // every lane of the consuming warp releases its reads
    }
    for (int par = 0; par < 2; ++par) {
      mbar_init(qfull(par), 1);
      mbar_init(mfull(par), NC * 32);  // every lane of every consumer arrives after its deposit
      mbar_init(tfree(par), 32);       // every lane of the merge warp, after reading the deposits
    }
    for (int q = 0; q < CQ; ++q) {
      mbar_init(cqfull(q), 1);
      mbar_init(cqempty(q), 1);
    }
    if (cl) mbar_init(clfull, p.nsplit * 32);  // every lane of every merge warp of the cluster
    *pop_ctr = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if (cl) cluster_sync_all();  // the leader's barrier is initialised before any remote arrival
  if (warp == 0 && quest_k == 0) {
    // Warm L2 with this CTA's first owned tile while the previous kernel drains (its tail
    // leaves HBM idle).  Only a hint: nothing is read from these lines before griddepcontrol.wait
    // below, and L2 is the point of coherence, so a row the previous kernel rewrites is seen.
    const int fu = p.units / (int)gridDim.x;
    if (fu > 0) {
      const int unit0 = blockIdx.x * fu;
      // about an eighth of the CTA's owned tiles, 1..RAAS_PREFETCH_TILES (config 3, 12 owned
      // tiles: 2; config 4 and the small budgets, 4-8: 1; L = 4096 / 8192, 24 / 48: 3 / 4;
      // measured per config, see profiles/r01_schedule_study.md)
      const int npf = min(RAAS_PREFETCH_TILES, max(1, (fu * p.nsplit + 4) / 8));
      for (int pg = lane; pg < min(npf * p.split_pages, fu * p.C); pg += 32)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                         p.kvstore + ((size_t)unit0 * p.C + pg) * p.pstr),  // unit-major
                     "r"(p.pstr * 2)
                     : "memory");
    }
  }
  // Early start (p.early: the host saw that the previous kernel of the stream
  // is not this handle's decode step): this handle's state was written by a kernel that
  // completed before the previous one could trigger us, so the producer reads its first tile's
  // metadata and issues that tile's first page copies BEFORE griddepcontrol.wait (below); only
  // the step's inputs (q, k_new, v_new) and every store wait for the previous kernel.
  const bool early = p.early != 0;  // hybrid: only its selection-independent pages (producer)
  if (!(early && warp == 0)) {
    pdl_wait();  // everything above overlapped the previous kernel; state reads start here
    pdl_launch_dependents();
  }
  const long long t_start = dbg_clock();
#ifdef RAAS_DBG_TIMING
  if (threadIdx.x == 0) g_raas_dbg[blockIdx.x][12] = dbg_gtimer();
  if (threadIdx.x == 0 && blockIdx.x < 256) g_raas_tl[p.dbg_slot & 7][blockIdx.x][1] = dbg_gtimer();
#endif

  const int C = p.C, SP = p.split_pages, g = p.g;  // C: 16-row tiles (pages) per unit
  const int n_tiles = p.units * p.nsplit;
  const bool tok = (GEN || TOKD) && p.ep == 1;  // token-level RaaS (NEXT-3): metadata per row, tiles physical only

  // multi-consumer combine queue: the combine warp from the start, the consumers after END
  auto combine_loop = [&](uint32_t scratch) {
    for (;;) {
      int i = 0;
      if (lane == 0) i = atomicAdd(pop_ctr, 1);
      i = __shfl_sync(0xffffffffu, i, 0);
      const int q = i % CQ;
      RAAS_TIMED(4, mbar_wait(cqfull(q), (i / CQ) & 1));
      int entry = 0;
      if (lane == 0) entry = cq[q];
      entry = __shfl_sync(0xffffffffu, entry, 0);
      const bool outdone = entry >= 0 && (entry & CQ_OUTDONE);
      if (outdone && lane == 0) {  // the slot's LSE row -> this popper's scratch (the lane that
        // releases the slot does every read of it)
#pragma unroll
        for (int h = 0; h < MAX_GROUP; ++h)
          sts_f32(scratch + MAX_SPLITS * MAX_GROUP * 8 + 4 * h, lds_f32(lseq + 4 * (q * MAX_GROUP + h)));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(cqempty(q));  // the entry is read: the slot may be refilled
      if (entry < 0) break;
      const int unit = entry & ((1 << CQ_UNIT_BITS) - 1);
      const int nse_u = (entry >> CQ_UNIT_BITS) & CQ_NSE_MASK;
      // partials of other SMs: released by their merge warps' acq_rel counter increments and
      // acquired by our merge warp's (the same lane then pushes: mbarrier arrive = release.cta,
      // our wait = acquire.cta).  Causality order is transitive, so no further fence is needed;
      // the partials are read with ld.global.cg (L2, the point of coherence)
#ifdef RAAS_DBG_TIMING
      if (lane == 0 && unit < 4096) { g_raas_dbg_unit[unit][0] = blockIdx.x; g_raas_dbg_unit[unit][2] = dbg_gtimer(); }
#endif
      if constexpr (TOKD) combine_unit_tok<D>(p, unit, nse_u, scratch, lane);
      else        combine_unit<D, GEN, FM>(p, unit, nse_u, scratch, lane, outdone, cl, recv, clfull);
#ifdef RAAS_DBG_TIMING
      if (lane == 0 && unit < 4096) g_raas_dbg_unit[unit][3] = dbg_gtimer();
#endif
      __syncwarp();
    }
  };

  if (warp == 0) {
    // =============================== TMA producer ===============================
    const uint64_t pol = l2_evict_first_policy();
    int4 nplan = make_int4(0, 0, 0, 0);
    int ncnt = 0;
    // a tile covers the "attended page list" positions v in [split*SP, split*SP + SP): the
    // resident pages in index order, or, in the Quest-on-prefill hybrid (NEXT-4), the K
    // selected full prompt pages (from raas_qselect) followed by every page from nfull on
    int nphys = 0, nnatt = 0, nndep = 0;  // nndep: leading positions independent of the selection
    auto fetch = [&](int tl) {
      if (tl < n_tiles) {
        const int u = tl / p.nsplit, q0 = (tl - u * p.nsplit) * SP;
        nplan = __ldcg(p.plan + u);
        const int nf = quest_k > 0 ? p.nfull[u] : 0;
        const bool hyb = quest_k > 0 && nf > quest_k;
        const int v = q0 + lane;
        if (tok) {  // token slots: used slots are the prefix [0, z), so tile v holds z - 16v rows
          // (tokd: z excludes the new token, which the combine adds; an empty unit still
          // gets one empty tile so that its combine runs)
          nnatt = max((nplan.z + PAGE - 1) / PAGE, TOKD ? 1 : 0);
          nphys = v;
          ncnt = (lane < SP && v < nnatt) ? min(PAGE, nplan.z - PAGE * v) : 0;
        } else {
          // hybrid: the pages from nfull on first (they do not depend on this step's selection,
          // so an early start can issue them before griddepcontrol.wait), then the K selected
          // prompt pages, read only after the selection kernel (the previous grid) completed
          nnatt = hyb ? quest_k + nplan.z - nf : nplan.z;
          nndep = hyb ? nplan.z - nf : nnatt;
          nphys = !hyb ? v : v < nndep ? nf + v : v < nnatt ? __ldcg(p.vmap + (size_t)u * C + (v - nndep)) : 0;
          ncnt = (lane < SP && v < nnatt) ? __ldcg(p.cnt + (size_t)u * C + nphys) : 0;
        }
      }
    };
    // pages in batches, one lane per page: each lane waits for its stage, fills the stage
    // info and issues one 1-D bulk copy of the page (K rows then V rows, 16*D*4 contiguous
    // bytes, stored pre-swizzled in HBM so they land bank-conflict-free for ldmatrix).  A batch
    // never spans more than S positions: a parity wait must be at most one phase ahead of its
    // barrier.
    // Half a ring per batch: a batch's lanes reconverge after their empty waits, so a batch is
    // issued when its LAST stage frees; with whole-ring batches the ring drained before each
    // refill (config 4: 48.9 -> 46.7 us per launch with S / 2, config 3 -1.5 %; S / 4 and single
    // pages are slower; pre-issuing a whole ring at early start instead of one batch: no gain)
#ifndef RAAS_BATCH
    constexpr int BATCH = S / 2 < 32 ? S / 2 : 32;
#else
    constexpr int BATCH = RAAS_BATCH;
#endif
    auto issue_batch = [&](int i0, int nb, uint32_t jb, int unit, int n, int kt, int cntv, int physv,
                           int slot, int off) {
      const int c = __shfl_sync(0xffffffffu, cntv, (i0 + lane) & 31);
      const int page = __shfl_sync(0xffffffffu, physv, (i0 + lane) & 31);
      if (lane < nb) {
        const int i = i0 + lane;
        const uint32_t jj = jb + lane;
        const int s = (int)(jj % S);
        RAAS_TIMED(1, mbar_wait(empty(s), ((jj / S) & 1) ^ 1));
        // the tile the new token goes to, its row count and the row it is written to
        RAAS_CHK(unit >= 0 && unit < p.units && page >= 0 && page < C && c >= 0 && c <= PAGE, 0);
        const bool is_slot = TOKD ? false : tok ? page == (slot >> 4) : page == slot;
        const int patch = !is_slot ? -1 : (tok ? (slot & (PAGE - 1)) : off);
        sinfo[2 * s] = make_int4(unit, page, (is_slot && !tok) ? off + 1 : c, patch);
        sinfo[2 * s + 1] =
            make_int4(kt, (i < NC ? FLAG_FIRST : 0) | (i + NC >= n ? FLAG_LAST : 0), 0, 0);
        // the whole HBM page (pstr elements: K rows, V rows, and the tokd ts/start trailer or
        // the Quest min / max rows when the handle has one)
        mbar_arrive_expect_tx(full(s), p.pstr * 2);
        bulk_load_hint(ring + s * STAGE, p.kvstore + (size_t)(unit * C + page) * p.pstr,
                       p.pstr * 2, full(s), pol);
      }
      __syncwarp();
    };
    TileSched sched(p.units, p.nsplit, gridDim.x, blockIdx.x, cl);
    bool owned = false, owned_next = false;
    int tile = sched.next(p.sched, lane, owned);
    if (tile >= 0) fetch(tile);
    uint32_t j = 0;
    int k = 0;
    int pre = 0;  // pages of the first tile issued before griddepcontrol.wait (early start)
    if (early) {
      if (tile >= 0) {
        const int unit = tile / p.nsplit, p0 = (tile - unit * p.nsplit) * SP;
        const int n = min(p0 + SP, nnatt) - p0;
        if (n > 0) {
          // the whole first tile when the ring holds it (16-page tiles: small budgets, B = 1;
          // -1 % there), else one batch (32-page tiles: a second batch early cost config 4 +0.6 %)
          pre = RAAS_PRE > 0 ? min(n, RAAS_PRE < S ? RAAS_PRE : S) : (n <= S ? n : min(n, BATCH));
          // hybrid: only the positions before nndep are final before the wait
          if (quest_k > 0) pre = max(0, min(pre, nndep - p0));
          if (pre > 0) issue_batch(0, pre, 0, unit, n, 0, ncnt, nphys, nplan.x, nplan.y & 0xffff);
        }
      }
      pdl_wait();
      pdl_launch_dependents();
      if (quest_k > 0 && tile >= 0) fetch(tile);  // the selected pages of the first tile, now final
    }
    while (tile >= 0) {
      const int unit = tile / p.nsplit, split = tile - unit * p.nsplit;
      const int4 pl = nplan;
      const int cntv = ncnt, physv = nphys, natt = nnatt;
      // next tile (and its metadata, in flight while this tile is issued)
      const int tile_next = sched.next(p.sched, lane, owned_next);
      if (tile_next >= 0) fetch(tile_next);
      const bool owned_cur = owned;
      tile = tile_next;  // loop-carried; the body below uses unit/split/owned_cur
      owned = owned_next;
      const int p0 = split * SP;
      const int n = min(p0 + SP, natt) - p0;
      if (n <= 0) {  // pages not yet allocated (fill phase)
        // cluster schedule: the leader expects an arrival from every CTA of the cluster; an
        // empty split publishes nothing (its combine folds only the nse non-empty splits)
        if (cl) mbar_arrive_remote(mapa(clfull, 0));
        continue;
      }
      const int slot = pl.x, off = pl.y & 0xffff;
      // align the tile to the consumer count: page i of a tile is always consumed by warp
      // i % NC, so the split's arithmetic does not depend on the schedule (determinism)
      for (; j % NC != 0; ++j) {
        const int s = (int)(j % S);
        mbar_wait(empty(s), ((j / S) & 1) ^ 1);
        if (lane == 0) {
          sinfo[2 * s + 1] = make_int4(0, FLAG_SKIP, 0, 0);
          mbar_arrive(full(s));
        }
        __syncwarp();
      }
      const int par = k & 1;
      RAAS_TIMED(0, mbar_wait(tfree(par), ((k >> 1) & 1) ^ 1));  // tile k-2 merged: slots free
      if (lane == 0) {
        tinfo[3 * par] = make_int4(unit, split, (natt + SP - 1) / SP, n);
        tinfo[3 * par + 1] = make_int4((int)j, 0, owned_cur ? 1 : 0, 0);
        if constexpr (TOKD) {  // deferred decisions: npin, pending flag, their time stamp (t - 1)
          tinfo[3 * par + 2] = make_int4(__ldg(p.npin + unit), pl.y, pl.w - 1, 0);
          mbar_arrive_expect_tx(qfull(par), 2 * g * D * 2 + 32);
          bulk_load(qpb + par * Lay::QPBUF, p.q_prev + (size_t)unit * g * D, g * D * 2, qfull(par));
          bulk_load(qpb + par * Lay::QPBUF + Lay::QBUF, p.lse_prev + (size_t)unit * 8, 32, qfull(par));
        } else {
          mbar_arrive_expect_tx(qfull(par), g * D * 2);
        }
        bulk_load(qbuf + par * Lay::QBUF, p.q + (size_t)unit * g * D, g * D * 2, qfull(par));
        if (n < NC) mbar_arrive_cnt(mfull(par), (NC - n) * 32);  // warps with no page here
      }
      // the first tile's first batch may already be in flight (early start)
      if (pre > 0) j += pre;
      for (int i0 = pre; i0 < n; i0 += BATCH) {
        const int nb = min(BATCH, n - i0);
        issue_batch(i0, nb, j, unit, n, k, cntv, physv, slot, off);
        j += nb;
      }
      pre = 0;
      ++k;
    }
    for (int e = 0; e < NC; ++e, ++j) {  // one END sentinel per consumer
      const int s = (int)(j % S);
      mbar_wait(empty(s), ((j / S) & 1) ^ 1);
      if (lane == 0) {
        sinfo[2 * s + 1] = make_int4(0, FLAG_END, 0, 0);
        mbar_arrive(full(s));
      }
      __syncwarp();
    }
    const int par = k & 1;  // END for the merge warp
    mbar_wait(tfree(par), ((k >> 1) & 1) ^ 1);
    if (lane == 0) {
      tinfo[3 * par + 1] = make_int4(0, FLAG_END, 0, 0);
      mbar_arrive_cnt(mfull(par), NC * 32);
    }
    dbg_add(8, t_start);
#ifdef RAAS_DBG_TIMING
    if (lane == 0) g_raas_dbg[blockIdx.x][13] = dbg_gtimer();
    if (lane == 0 && blockIdx.x < 256) g_raas_tl[p.dbg_slot & 7][blockIdx.x][2] = dbg_gtimer();
#endif
  } else if (warp == 1) {
    // ============================ merge (per tile) ============================
    const int r = lane >> 2, qd = lane & 3;
    int npush = 0;
    // running merge of the current owned unit's splits (heads 2qd, 2qd+1 of this lane)
    float rm0 = -INFINITY, rm1 = -INFINITY, rl0 = 0.f, rl1 = 0.f, racc[KS * 4];
#pragma unroll
    for (int i = 0; i < KS * 4; ++i) racc[i] = 0.f;
    float lse0 = 0.f, lse1 = 0.f;  // pushed with an outdone unit
    auto push = [&](int unit) {  // hand a finished unit (or -1 = END) to the combine warp
#ifdef RAAS_DBG_TIMING
      if (lane == 0 && unit >= 0 && (unit & ((1 << CQ_UNIT_BITS) - 1)) < 4096) g_raas_dbg_unit[unit & ((1 << CQ_UNIT_BITS) - 1)][1] = dbg_gtimer();
#endif
      const int q = npush % CQ;
      RAAS_TIMED(7, mbar_wait(cqempty(q), ((npush / CQ) & 1) ^ 1));
      const bool od = unit >= 0 && (unit & CQ_OUTDONE);
      float lv[MAX_GROUP];  // the unit's LSE per head, gathered to lane 0 (head h: lane h / 2)
#pragma unroll
      for (int h = 0; h < MAX_GROUP; ++h) lv[h] = __shfl_sync(0xffffffffu, (h & 1) ? lse1 : lse0, h >> 1);
      if (lane == 0) {
        if (od) {
#pragma unroll
          for (int h = 0; h < MAX_GROUP; ++h) sts_f32(lseq + 4 * (q * MAX_GROUP + h), lv[h]);
        }
        cq[q] = unit;
        mbar_arrive(cqfull(q));
      }
      __syncwarp();
      ++npush;
    };
    for (int k = 0;; ++k) {
      const int par = k & 1;
      RAAS_TIMED(2, mbar_wait(mfull(par), (k >> 1) & 1));
      const int4 t0 = tinfo[3 * par], t1 = tinfo[3 * par + 1];
      if (t1.y & FLAG_END) {
        for (int e = 0; e < Lay::NPOP; ++e) push(-1);
        break;
      }
      const int unit = t0.x, split = t0.y, nse = t0.z, n = t0.w, J = t1.x, owned = t1.z;
      RAAS_CHK(unit >= 0 && unit < p.units && split >= 0 && split < nse && nse <= p.nsplit &&
                   n > 0 && n <= p.split_pages, 2);
      const int nw = min(n, NC);
      float acc[KS * 4];
#pragma unroll
      for (int i = 0; i < KS * 4; ++i) acc[i] = 0.f;
      float M0 = -INFINITY, M1 = -INFINITY, L0 = 0.f, L1 = 0.f;
      for (int i = 0; i < nw; ++i) {
        const uint32_t dep = merge + ((par % Lay::NDEP) * NC + (J + i) % NC) * Lay::DEPOSIT + 4 * lane;
        M0 = fmaxf(M0, lds_f32(dep + 128 * (KS * 4 + 0)));
        M1 = fmaxf(M1, lds_f32(dep + 128 * (KS * 4 + 1)));
      }
      const float M0b = M0 == -INFINITY ? 0.f : M0, M1b = M1 == -INFINITY ? 0.f : M1;  // empty tile
      for (int i = 0; i < nw; ++i) {
        const uint32_t dep = merge + ((par % Lay::NDEP) * NC + (J + i) % NC) * Lay::DEPOSIT + 4 * lane;
        const float s0 = fast_exp2(lds_f32(dep + 128 * (KS * 4 + 0)) - M0b);
        const float s1 = fast_exp2(lds_f32(dep + 128 * (KS * 4 + 1)) - M1b);
        L0 += s0 * lds_f32(dep + 128 * (KS * 4 + 2));
        L1 += s1 * lds_f32(dep + 128 * (KS * 4 + 3));
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) {
          acc[4 * mt + 0] += s0 * lds_f32(dep + 128 * (4 * mt + 0));
          acc[4 * mt + 1] += s1 * lds_f32(dep + 128 * (4 * mt + 1));
          acc[4 * mt + 2] += s0 * lds_f32(dep + 128 * (4 * mt + 2));
          acc[4 * mt + 3] += s1 * lds_f32(dep + 128 * (4 * mt + 3));
        }
      }
      int4 ck = make_int4(-1, -1, -1, 0);  // tokd: the tile's victim candidate (min key)
      if constexpr (TOKD) {
        if (lane < nw) {
          const uint32_t ca = cand + (par * NC + (J + lane) % NC) * 16;
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(ck.x), "=r"(ck.y), "=r"(ck.z), "=r"(ck.w) : "r"(ca));
        }
        unsigned long long key = (static_cast<unsigned long long>(static_cast<uint32_t>(ck.y)) << 32) |
                                 static_cast<uint32_t>(ck.x);
        const unsigned long long kmin = warp_min_u64(key);
        const unsigned hit = __ballot_sync(0xffffffffu, key == kmin);
        ck.z = __shfl_sync(0xffffffffu, ck.z, __ffs(hit) - 1);
        ck.x = static_cast<int>(static_cast<uint32_t>(kmin));
        ck.y = static_cast<int>(static_cast<uint32_t>(kmin >> 32));
      }
      __syncwarp();
      mbar_arrive(tfree(par));  // deposits / q / info of tile k consumed (each lane's reads)
      if (!TOKD && owned) {
        // an owned unit's splits arrive here in order on this CTA: fold the tile into the
        // running merge; after the last split write out and hand the LSE to the combine
        if (split == 0) {
          rm0 = rm1 = -INFINITY;
          rl0 = rl1 = 0.f;
#pragma unroll
          for (int i = 0; i < KS * 4; ++i) racc[i] = 0.f;
        }
        float mn0, fa0, fb0, mn1, fa1, fb1;
        merge_factors(rm0, M0, mn0, fa0, fb0);
        merge_factors(rm1, M1, mn1, fa1, fb1);
        rl0 = fmaf(rl0, fa0, __fmul_rn(L0, fb0));
        rl1 = fmaf(rl1, fa1, __fmul_rn(L1, fb1));
        rm0 = mn0;
        rm1 = mn1;
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) {
          racc[4 * mt + 0] = fmaf(racc[4 * mt + 0], fa0, __fmul_rn(acc[4 * mt + 0], fb0));
          racc[4 * mt + 1] = fmaf(racc[4 * mt + 1], fa1, __fmul_rn(acc[4 * mt + 1], fb1));
          racc[4 * mt + 2] = fmaf(racc[4 * mt + 2], fa0, __fmul_rn(acc[4 * mt + 2], fb0));
          racc[4 * mt + 3] = fmaf(racc[4 * mt + 3], fa1, __fmul_rn(acc[4 * mt + 3], fb1));
        }
        if (split == nse - 1) {
          const float inv0 = 1.f / rl0, inv1 = 1.f / rl1;
          lse0 = rm0 + log2f(rl0);
          lse1 = rm1 + log2f(rl1);
          __nv_bfloat16* o0 = p.out + (size_t)(unit * g + 2 * qd) * D + r;
          __nv_bfloat16* o1 = o0 + D;
#pragma unroll
          for (int mt = 0; mt < KS; ++mt) {
            if (2 * qd < g) {
              o0[16 * mt] = __float2bfloat16_rn(racc[4 * mt + 0] * inv0);
              o0[16 * mt + 8] = __float2bfloat16_rn(racc[4 * mt + 2] * inv0);
            }
            if (2 * qd + 1 < g) {
              o1[16 * mt] = __float2bfloat16_rn(racc[4 * mt + 1] * inv1);
              o1[16 * mt + 8] = __float2bfloat16_rn(racc[4 * mt + 3] * inv1);
            }
          }
          push(unit | nse << CQ_UNIT_BITS | CQ_OWNED | CQ_OUTDONE);
        }
        continue;
      }
      if (cl) {
        // cluster schedule: this split's partial goes straight into the leader's receive slot
        // (distributed shared memory stores), then every lane arrives on the leader's barrier
        // (release at cluster scope orders its stores before the leader's acquire)
        const uint32_t slot = mapa(recv + split * Lay::RECV_SLOT, 0);
        if (lane < 4) {
          if (2 * qd < g) {
            st_dsmem_f32(slot + 8 * (2 * qd), M0);
            st_dsmem_f32(slot + 8 * (2 * qd) + 4, L0);
          }
          if (2 * qd + 1 < g) {
            st_dsmem_f32(slot + 8 * (2 * qd + 1), M1);
            st_dsmem_f32(slot + 8 * (2 * qd + 1) + 4, L1);
          }
        }
        const uint32_t pa0 = slot + PUB_ACC_OFF + ((2 * qd) * D + r) * 4, pa1 = pa0 + D * 4;
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) {
          if (2 * qd < g) { st_dsmem_f32(pa0 + 64 * mt, acc[4 * mt + 0]); st_dsmem_f32(pa0 + 64 * mt + 32, acc[4 * mt + 2]); }
          if (2 * qd + 1 < g) { st_dsmem_f32(pa1 + 64 * mt, acc[4 * mt + 1]); st_dsmem_f32(pa1 + 64 * mt + 32, acc[4 * mt + 3]); }
        }
        mbar_arrive_remote(mapa(clfull, 0));
        if (split == 0) push(unit | nse << CQ_UNIT_BITS);  // split 0 is the leader's (rank 0)
        continue;
      }
      // publish the tile's split-K partial (m, l, acc) in the C-fragment layout
      const int pbase = (unit * p.nsplit + split) * g;
      if (TOKD && lane == 0) p.part_key[unit * p.nsplit + split] = ck;
      if (lane < 4) {
        if (2 * qd < g) p.part_ml[pbase + 2 * qd] = make_float2(M0, L0);
        if (2 * qd + 1 < g) p.part_ml[pbase + 2 * qd + 1] = make_float2(M1, L1);
      }
      float* pa0 = p.part_acc + (size_t)(pbase + 2 * qd) * D + r;
      float* pa1 = pa0 + D;
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        if (2 * qd < g) { pa0[16 * mt] = acc[4 * mt + 0]; pa0[16 * mt + 8] = acc[4 * mt + 2]; }
        if (2 * qd + 1 < g) { pa1[16 * mt] = acc[4 * mt + 1]; pa1[16 * mt + 8] = acc[4 * mt + 3]; }
      }
      __syncwarp();
      if (owned) {  // every split of the unit is ours and in order: no cross-CTA counter
        if (split == nse - 1) push(unit | nse << CQ_UNIT_BITS | CQ_OWNED);
      } else {
        int old = 0;  // release our partial / acquire the others' (gpu scope, cumulative)
        if (lane == 0) old = atom_add_acq_rel_gpu(p.counter + unit, 1);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old == nse - 1) push(unit | nse << CQ_UNIT_BITS);  // the unit's last split
      }
    }
    dbg_add(9, t_start);
  } else if (warp == 2) {
    // ============================ combine (per unit) ============================
    if (cl) {
      // cluster schedule: only the leader combines, one unit, with its metadata loaded now (the
      // previous step's state, final once griddepcontrol.wait returned above) so none of its
      // loads sits on the combine's critical path
      if (cluster_ctarank() == 0) {
        const int unit = blockIdx.x / p.nsplit;
        ClMeta cm;
        cm.pl = __ldcg(p.plan + unit);
        cm.npin = __ldg(p.npin + unit);
#pragma unroll
        for (int i = 0; i < CLM; ++i) {
          const int pg = 32 * i + lane;
          cm.ts[i] = pg < C ? __ldcg(p.ts + (size_t)unit * C + pg) : 0;
          cm.st[i] = pg < C ? __ldcg(p.start + (size_t)unit * C + pg) : 0;
        }
        int i = 0;
        if (lane == 0) i = atomicAdd(pop_ctr, 1);  // index 0: the unit (the consumers never pop)
        i = __shfl_sync(0xffffffffu, i, 0);
        mbar_wait(cqfull(i % CQ), (i / CQ) & 1);
        int entry = 0;
        if (lane == 0) entry = cq[i % CQ];
        entry = __shfl_sync(0xffffffffu, entry, 0);
        __syncwarp();
        if (lane == 0) mbar_arrive(cqempty(i % CQ));
        if (entry >= 0) {
          const int unit_e = entry & ((1 << CQ_UNIT_BITS) - 1);
#ifdef RAAS_DBG_TIMING
          if (lane == 0 && unit_e < 4096) { g_raas_dbg_unit[unit_e][0] = blockIdx.x; g_raas_dbg_unit[unit_e][2] = dbg_gtimer(); }
#endif
          combine_unit_cl<D>(p, unit_e, (entry >> CQ_UNIT_BITS) & CQ_NSE_MASK, scr, lane, recv,
                             recv + p.nsplit * Lay::RECV_SLOT, clfull, cm);
#ifdef RAAS_DBG_TIMING
          if (lane == 0 && unit_e < 4096) g_raas_dbg_unit[unit_e][3] = dbg_gtimer();
#endif
        }
      }
    } else {
      combine_loop(scr);
    }
    dbg_add(10, t_start);
#ifdef RAAS_DBG_TIMING
    if (lane == 0) g_raas_dbg[blockIdx.x][14] = dbg_gtimer();
#endif
  } else {
    // ================================ consumers ================================
    const int w = warp - 3;
    const int r = lane >> 2, qd = lane & 3;   // C-fragment row (token) / column pair (head)
    const int mi = lane >> 3, ri = lane & 7;  // ldmatrix matrix / row supplied by this lane
    float acc[KS][4];
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    uint32_t qb[KS][2];
    // tokd: previous step's q fragments and LSE, its pending-decision info, the tile's running
    // victim candidate, and this warp's decision counters (kept on the qd == 0 lanes)
    uint32_t qp[KS][2];
    float lp0 = INFINITY, lp1 = INFINITY;
    int npin_t = 0, pend_t = 0, tm1 = 0, cslot = -1, n_dec = 0, n_stamp = 0;
    unsigned long long ckey = ~0ull;
#pragma unroll
    for (int mt = 0; mt < KS; ++mt) {
      acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
      qb[mt][0] = qb[mt][1] = 0u;
    }
    for (uint32_t j = w;; j += NC) {
      const int s = (int)(j % S);
      RAAS_TIMED(5, mbar_wait(full(s), (j / S) & 1));
      const int4 i0 = sinfo[2 * s], i1 = sinfo[2 * s + 1];
      const int flags = i1.y;
      if (flags & FLAG_END) {
        if constexpr (TOKD) {  // deferred decisions taken by this warp over the whole launch
          n_dec = warp_sum_i(n_dec);
          n_stamp = warp_sum_i(n_stamp);
          if (lane == 0 && n_dec) {
            atomicAdd(p.stats + 0, (unsigned long long)n_stamp);
            atomicAdd(p.stats + 1, (unsigned long long)n_dec);
          }
        }
        if constexpr (Lay::JOIN) {
          if (!cl) combine_loop(ring + s * STAGE);  // join the tail's combines
        }
        break;
      }
      if (flags & FLAG_SKIP) {
        __syncwarp();
        mbar_arrive(empty(s));
        continue;
      }
      const int unit = i0.x, page = i0.y, cnt = i0.z, patch = i0.w, k = i1.x, par = k & 1;
      RAAS_CHK(unit >= 0 && unit < p.units && page >= 0 && page < C && cnt >= 0 && cnt <= PAGE &&
                   patch >= -1 && patch < PAGE, 1);
      const uint32_t kb = ring + s * STAGE, vb = kb + TILE;

      if (flags & FLAG_FIRST) {  // fresh softmax state; this unit's q fragments from smem
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
        m0 = m1 = -INFINITY;
        l0 = l1 = 0.f;
        RAAS_TIMED(6, mbar_wait(qfull(par), (k >> 1) & 1));
        const uint32_t qrow = qbuf + par * Lay::QBUF + r * D * 2 + qd * 4;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          qb[ks][0] = r < g ? lds_u32(qrow + ks * 32) : 0u;       // d = 16ks + 2qd, +1
          qb[ks][1] = r < g ? lds_u32(qrow + ks * 32 + 16) : 0u;  // d = 16ks + 8 + 2qd, +1
        }
        if constexpr (TOKD) {
          const int4 ti = tinfo[3 * par + 2];
          npin_t = ti.x;
          pend_t = ti.y;
          tm1 = ti.z;
          const uint32_t qprow = qpb + par * Lay::QPBUF + r * D * 2 + qd * 4;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            qp[ks][0] = r < g ? lds_u32(qprow + ks * 32) : 0u;
            qp[ks][1] = r < g ? lds_u32(qprow + ks * 32 + 16) : 0u;
          }
          const uint32_t lpa = qpb + par * Lay::QPBUF + Lay::QBUF;
#ifdef RAAS_DBG_TOKD_GLOBAL
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            if (r < g) {
              const uint32_t* gq = reinterpret_cast<const uint32_t*>(p.q_prev + ((size_t)unit * g + r) * D);
              if (qp[ks][0] != __ldcg(gq + ks * 8 + qd) || qp[ks][1] != __ldcg(gq + ks * 8 + 4 + qd)) {
                if (atomicOr(p.status, 8u) == 0u) {
                  g_tokd_dbg[0] = unit; g_tokd_dbg[1] = page; g_tokd_dbg[2] = k; g_tokd_dbg[3] = par;
                  g_tokd_dbg[4] = tm1; g_tokd_dbg[5] = pend_t; g_tokd_dbg[6] = (int)qp[ks][0];
                  g_tokd_dbg[7] = (int)__ldcg(gq + ks * 8 + qd); g_tokd_dbg[8] = blockIdx.x; g_tokd_dbg[9] = w;
                  g_tokd_dbg[10] = r; g_tokd_dbg[11] = ks; g_tokd_dbg[12] = flags;
                }
              }
            }
          }
          lp0 = 2 * qd < g ? __ldcg(p.lse_prev + unit * 8 + 2 * qd) : INFINITY;
          lp1 = 2 * qd + 1 < g ? __ldcg(p.lse_prev + unit * 8 + 2 * qd + 1) : INFINITY;
          if (lp0 != (2 * qd < g ? lds_f32(lpa + 8 * qd) : INFINITY)) atomicOr(p.status, 4u);
#else
          lp0 = 2 * qd < g ? lds_f32(lpa + 8 * qd) : INFINITY;  // head 2qd (+inf: not a head)
          lp1 = 2 * qd + 1 < g ? lds_f32(lpa + 8 * qd + 4) : INFINITY;
#endif
          ckey = ~0ull;
          cslot = -1;
        }
      }

      if (patch >= 0) {  // a2: the new token's K/V into row `patch` (smem tile + HBM store)
        constexpr int NCH = D / 8;
        if (lane < 2 * NCH) {
          const bool isv = lane >= NCH;
          const int ch = isv ? lane - NCH : lane;
          const uint4 val = __ldg(reinterpret_cast<const uint4*>(
                                      (isv ? p.v_new : p.k_new) + (size_t)unit * D) + ch);
          const int phys = ch ^ (patch & 7);  // pre-swizzled page layout (see raas_kernels.cuh)
          const uint32_t sa = (isv ? vb : kb) + patch * ROW + (phys << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(sa), "r"(val.x),
                       "r"(val.y), "r"(val.z), "r"(val.w)
                       : "memory");
          *reinterpret_cast<uint4*>(p.kvstore + (size_t)(unit * C + page) * p.pstr +
                                    ((isv ? PAGE : 0) + patch) * D + phys * 8) = val;
          if ((GEN || (FM & F_QUEST)) && score_mode == 1 && !isv) {
            // the page's per-channel min / max rows (Quest representative keys, maintained on
            // write): a fresh page (row 0) restarts them from the new key
            const uint32_t ta = kb + 2 * TILE + ch * 16;
            uint4 mn = val, mx = val;
            if (patch > 0) {
              uint4 omn, omx;
              asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(omn.x), "=r"(omn.y), "=r"(omn.z), "=r"(omn.w) : "r"(ta));
              asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(omx.x), "=r"(omx.y), "=r"(omx.z), "=r"(omx.w) : "r"(ta + 2 * D));
              asm("min.bf16x2 %0, %0, %1;" : "+r"(mn.x) : "r"(omn.x));
              asm("min.bf16x2 %0, %0, %1;" : "+r"(mn.y) : "r"(omn.y));
              asm("min.bf16x2 %0, %0, %1;" : "+r"(mn.z) : "r"(omn.z));
              asm("min.bf16x2 %0, %0, %1;" : "+r"(mn.w) : "r"(omn.w));
              asm("max.bf16x2 %0, %0, %1;" : "+r"(mx.x) : "r"(omx.x));
              asm("max.bf16x2 %0, %0, %1;" : "+r"(mx.y) : "r"(omx.y));
              asm("max.bf16x2 %0, %0, %1;" : "+r"(mx.z) : "r"(omx.z));
              asm("max.bf16x2 %0, %0, %1;" : "+r"(mx.w) : "r"(omx.w));
            }
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta), "r"(mn.x), "r"(mn.y),
                         "r"(mn.z), "r"(mn.w) : "memory");
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta + 2 * D), "r"(mx.x),
                         "r"(mx.y), "r"(mx.z), "r"(mx.w) : "memory");
            __nv_bfloat16* tg = p.kvstore + (size_t)(unit * C + page) * p.pstr + 2 * PAGE * D;
            *reinterpret_cast<uint4*>(tg + ch * 8) = mn;
            *reinterpret_cast<uint4*>(tg + D + ch * 8) = mx;
          }
          fence_proxy_async_smem();  // before the stage is refilled by TMA
        }
        __syncwarp();
      }

#ifdef RAAS_DBG_NOCOMPUTE  // pipeline-ceiling experiment: consume without computing
      __syncwarp();
      mbar_arrive(empty(s));
      if (flags & FLAG_LAST) {
        __syncwarp();
        mbar_arrive(mfull(par));  // each lane releases its own deposit writes
      }
      continue;
#endif
      // ---- a3/a4: S^T = K_page Q^T (M = 16 tokens, N = 8 heads, K = D) ----
      float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
      float e0[4] = {0.f, 0.f, 0.f, 0.f}, e1[4] = {0.f, 0.f, 0.f, 0.f};  // tokd: K q_prev^T
      const bool dec = TOKD && pend_t;
      {
        const uint32_t krow = kb + (ri + 8 * (mi & 1)) * ROW;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          uint32_t a[4];
          const int chunk = 2 * ks + (mi >> 1);
          ldsm_x4(krow + ((chunk ^ ri) << 4), a);
          if (ks & 1) mma_bf16_16816(c1, a, qb[ks][0], qb[ks][1]);
          else        mma_bf16_16816(c0, a, qb[ks][0], qb[ks][1]);
          if (TOKD && dec) {
            if (ks & 1) mma_bf16_16816(e1, a, qp[ks][0], qp[ks][1]);
            else        mma_bf16_16816(e0, a, qp[ks][0], qp[ks][1]);
          }
        }
      }
      int tsr[2] = {0, 0}, str2[2] = {0, 0};  // tokd: this lane's rows' ts / start (trailer)
      if constexpr (TOKD) {
        const uint32_t tb = kb + 2 * TILE;
        tsr[0] = (int)lds_u32(tb + 4 * r);
        tsr[1] = (int)lds_u32(tb + 4 * (r + 8));
        str2[0] = (int)lds_u32(tb + 64 + 4 * r);
        str2[1] = (int)lds_u32(tb + 64 + 4 * (r + 8));
      }
      // V^T fragments now, so the stage can be handed back to the producer before the softmax
      // and PV math: the ring slot is held ~100 cycles instead of a whole page's compute
      uint32_t va[KS][4];
      {
        const uint32_t vrow = vb + (ri + 8 * (mi >> 1)) * ROW;
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) {
          const int chunk = 2 * mt + (mi & 1);
          ldsm_x4_t(vrow + ((chunk ^ ri) << 4), va[mt]);
        }
      }
      auto release_stage = [&]() {
        uint32_t dep = 0;  // consume every fragment: the ldmatrix reads have completed
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) dep ^= va[mt][0] ^ va[mt][1] ^ va[mt][2] ^ va[mt][3];
        if constexpr (TOKD) dep ^= tsr[0] ^ tsr[1] ^ str2[0] ^ str2[1];
        asm volatile("" ::"r"(dep));
        __syncwarp();
        mbar_arrive(empty(s));  // stage free for the producer
      };
#ifdef RAAS_DBG_HOLD  // sensitivity probe: the stage held longer before its release
      {
        const long long t0 = clock64();
        while (clock64() - t0 < RAAS_DBG_HOLD) {
        }
      }
#endif
      if (score_mode == 0) release_stage();
      if constexpr (TOKD) {
        // deferred a6 (step t-1's stamps, PAPER.md :98-100 at token level) and a7 candidates:
        // row r and r + 8 of this tile, decision x = max_h (s'_h - LSE'_h) > log2(alpha)
        const int rows[2] = {r, r + 8};
        float xr[2];
        xr[0] = fmaxf((e0[0] + e1[0]) * p.scale_log2 - lp0, (e0[1] + e1[1]) * p.scale_log2 - lp1);
        xr[1] = fmaxf((e0[2] + e1[2]) * p.scale_log2 - lp0, (e0[3] + e1[3]) * p.scale_log2 - lp1);
        unsigned long long kmin = ~0ull;
        int rmin = 0;
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
          float x = xr[hr];
          x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 1));
          x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 2));
          const int row = rows[hr], e = page * PAGE + row;
          const bool valid = row < cnt && e >= npin_t;
          int tsv = tsr[hr];
          const int stv = str2[hr];
          const bool stamp = dec && valid && x > p.log2_alpha;  // strict (D3)
          if (stamp) tsv = tm1;
          if (qd == 0) {
            n_dec += (dec && valid) ? 1 : 0;
            n_stamp += stamp ? 1 : 0;
            if (stamp) {
              p.ts[(size_t)unit * p.Ce + e] = tm1;
              reinterpret_cast<int32_t*>(p.kvstore + (size_t)(unit * C + page) * p.pstr + 2 * PAGE * D)[row] = tm1;
            }
          }
          const unsigned long long key = valid ? cand_key(tsv, stv) : ~0ull;
          if (key < kmin) { kmin = key; rmin = row; }
        }
        // this lane's running minimum over its rows of the tile (reduced over the warp once,
        // at the tile's last page; keys are unique: start positions differ)
        if (kmin < ckey) {
          ckey = kmin;
          cslot = page * PAGE + rmin;
        }
      }
      float s0 = (c0[0] + c1[0]) * p.scale_log2, s1 = (c0[1] + c1[1]) * p.scale_log2;
      float s2 = (c0[2] + c1[2]) * p.scale_log2, s3 = (c0[3] + c1[3]) * p.scale_log2;
      if (r >= cnt) s0 = s1 = -INFINITY;
      if (r + 8 >= cnt) s2 = s3 = -INFINITY;
      float pm0 = fmaxf(s0, s2), pm1 = fmaxf(s1, s3);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        pm0 = fmaxf(pm0, __shfl_xor_sync(0xffffffffu, pm0, o));
        pm1 = fmaxf(pm1, __shfl_xor_sync(0xffffffffu, pm1, o));
      }
      float sc0 = pm0, sc1 = pm1;  // the page score the stamp will use (log2 domain)
      if (score_mode == 1) {
        // Quest's representative-key bound (PAPER.md :147-151, :362; reading D22): per channel
        // c, max(q_c min_c, q_c max_c) over the page's valid keys, summed over c.  Lane l owns
        // channels [l*CQ, (l+1)*CQ).  The per-channel min / max rows ("a representative key
        // (K) for each page", :147) are maintained on write and arrive with the page (+2 rows
        // per 32 K/V rows of bytes), so no key row is scanned here.
        constexpr int CQL = D / 32;
        const int c0 = lane * CQL;
        uint32_t mnp[CQL / 2], mxp[CQL / 2];  // packed bf16x2 min / max (exact)
        {
          const uint32_t a = kb + 2 * TILE + c0 * 2;
          if constexpr (CQL == 4) {
            asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(mnp[0]), "=r"(mnp[1]) : "r"(a));
            asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(mxp[0]), "=r"(mxp[1]) : "r"(a + 2 * D));
          } else {
            mnp[0] = lds_u32(a);
            mxp[0] = lds_u32(a + 2 * D);
          }
        }
        release_stage();  // the page's rows are no longer needed
        float mnv[CQL], mxv[CQL];
#pragma unroll
        for (int i = 0; i < CQL; ++i) {
          mnv[i] = __uint_as_float((i & 1) ? (mnp[i >> 1] & 0xffff0000u) : (mnp[i >> 1] << 16));
          mxv[i] = __uint_as_float((i & 1) ? (mxp[i >> 1] & 0xffff0000u) : (mxp[i >> 1] << 16));
        }
        const uint32_t qh0 = qbuf + par * Lay::QBUF + c0 * 2;
        float v[MAX_GROUP];
#pragma unroll
        for (int h = 0; h < MAX_GROUP; ++h) {
          v[h] = 0.f;
          if (h < g) {
            uint32_t w[CQL / 2];
            if constexpr (CQL == 4) {
              asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(qh0 + h * D * 2));
            } else {
              w[0] = lds_u32(qh0 + h * D * 2);
            }
#pragma unroll
            for (int i = 0; i < CQL; ++i) {
              const float qv = __uint_as_float((i & 1) ? (w[i >> 1] & 0xffff0000u) : (w[i >> 1] << 16));
              v[h] += fmaxf(qv * mnv[i], qv * mxv[i]);
            }
          }
        }
        // transpose-reduce the 8 per-head partial sums over the warp (9 shuffles instead of
        // 8 x 5): afterwards lane l holds head ((l>>4)&1)*4 + ((l>>3)&1)*2 + ((l>>2)&1)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool hi = lane & 16;
          const float send = hi ? v[i] : v[i + 4], keep = hi ? v[i + 4] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const bool hi = lane & 8;
          const float send = hi ? v[i] : v[i + 2], keep = hi ? v[i + 2] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
        {
          const bool hi = lane & 4;
          const float send = hi ? v[0] : v[1], keep = hi ? v[1] : v[0];
          v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
        auto lane_of = [](int h) { return ((h >> 2) & 1) << 4 | ((h >> 1) & 1) << 3 | (h & 1) << 2; };
        sc0 = __shfl_sync(0xffffffffu, v[0], lane_of(2 * qd)) * p.scale_log2;
        sc1 = __shfl_sync(0xffffffffu, v[0], lane_of(2 * qd + 1)) * p.scale_log2;
      }
      if (tok) {  // a4, token level (§3.2): every row's logit per head (tokd: none, deferred)
        float* px = p.pmax + ((size_t)(unit * C + page) * PAGE + r) * g;
        if (!TOKD && r < cnt) {
          if (2 * qd < g) px[2 * qd] = s0;
          if (2 * qd + 1 < g) px[2 * qd + 1] = s1;
        }
        if (!TOKD && r + 8 < cnt) {
          if (2 * qd < g) px[8 * g + 2 * qd] = s2;
          if (2 * qd + 1 < g) px[8 * g + 2 * qd + 1] = s3;
        }
      } else if (cl) {  // cluster schedule: the page maxima go to the leader's shared memory
        if (lane < 4) {
          const uint32_t pa = mapa(recv + p.nsplit * Lay::RECV_SLOT + 4 * (page * g), 0);
          if (2 * qd < g) st_dsmem_f32(pa + 4 * (2 * qd), sc0);
          if (2 * qd + 1 < g) st_dsmem_f32(pa + 4 * (2 * qd + 1), sc1);
        }
      } else if (lane < 4) {  // a4: page score per head ("a single attention score per page", :147)
        float* pmx = p.pmax + (size_t)(unit * C + page) * g;
        if (2 * qd < g) pmx[2 * qd] = sc0;
        if (2 * qd + 1 < g) pmx[2 * qd + 1] = sc1;
      }
      const float mn0 = fmaxf(m0, pm0), mn1 = fmaxf(m1, pm1);
      // reference maxima: 0 while nothing is valid yet (an empty tile in the token mode)
      const float mb0 = mn0 == -INFINITY ? 0.f : mn0, mb1 = mn1 == -INFINITY ? 0.f : mn1;
      const float cr0 = fast_exp2(m0 - mb0), cr1 = fast_exp2(m1 - mb1);
      m0 = mn0;
      m1 = mn1;
      const float p0 = fast_exp2(s0 - mb0), p1 = fast_exp2(s1 - mb1);
      const float p2 = fast_exp2(s2 - mb0), p3 = fast_exp2(s3 - mb1);
      l0 = l0 * cr0 + (p0 + p2);
      l1 = l1 * cr1 + (p1 + p3);
      // rescale only when some head's running max moved (x * 1 = x: bitwise the same result)
      if (!__all_sync(0xffffffffu, cr0 == 1.f && cr1 == 1.f)) {
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) {
          acc[mt][0] *= cr0;
          acc[mt][1] *= cr1;
          acc[mt][2] *= cr0;
          acc[mt][3] *= cr1;
        }
      }
      // P^T as the B operand of O^T = V^T P^T: transpose the two 8x8 bf16 blocks in registers
      const uint32_t b0 = movmatrix_t(pack_bf16x2(p0, p1));
      const uint32_t b1 = movmatrix_t(pack_bf16x2(p2, p3));
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) mma_bf16_16816(acc[mt], va[mt], b0, b1);
#ifdef RAAS_DBG_DELAY  // sensitivity probe: extra consumer time per page (after the release)
      {
        const long long t0 = clock64();
        while (clock64() - t0 < RAAS_DBG_DELAY) {
        }
      }
#endif

      if (flags & FLAG_LAST) {  // deposit this warp's softmax state for the tile merge
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          l0 += __shfl_xor_sync(0xffffffffu, l0, o);
          l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        }
        if constexpr (Lay::NDEP == 1) {
          // single deposit buffer: tile k - 1's deposits must have been read by the merge warp
          // (tfree of tile k - 1 = phase (k - 1) >> 1 of tfree((k - 1) & 1))
          if (k > 0) RAAS_TIMED(3, mbar_wait(tfree((k - 1) & 1), ((k - 1) >> 1) & 1));
        }
        const uint32_t dep = merge + ((par % Lay::NDEP) * NC + w) * Lay::DEPOSIT + 4 * lane;
#pragma unroll
        for (int mt = 0; mt < KS; ++mt)
#pragma unroll
          for (int e = 0; e < 4; ++e) sts_f32(dep + 128 * (4 * mt + e), acc[mt][e]);
        sts_f32(dep + 128 * (KS * 4 + 0), m0);
        sts_f32(dep + 128 * (KS * 4 + 1), m1);
        sts_f32(dep + 128 * (KS * 4 + 2), l0);
        sts_f32(dep + 128 * (KS * 4 + 3), l1);
        if constexpr (TOKD) {  // the warp's minimum over its lanes' running minima
          unsigned long long wk = ckey;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long w2 = __shfl_xor_sync(0xffffffffu, wk, o);
            wk = w2 < wk ? w2 : wk;
          }
          const unsigned hit = __ballot_sync(0xffffffffu, ckey == wk);
          const int ws = __shfl_sync(0xffffffffu, cslot, __ffs(hit) - 1);
          ckey = wk;
          cslot = wk == ~0ull ? -1 : ws;
        }
        if (TOKD && lane == 0) {  // the tile's victim candidate of this warp
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(cand + (par * NC + w) * 16),
                       "r"(static_cast<uint32_t>(ckey)), "r"(static_cast<uint32_t>(ckey >> 32)),
                       "r"(cslot), "r"(0)
                       : "memory");
        }
        __syncwarp();
        mbar_arrive(mfull(par));  // each lane releases its own deposit writes
      }
    }
    dbg_add(11, t_start);
  }
  // the last CTA out resets the dynamic-schedule counter for the next launch (which reads it
  // only after griddepcontrol.wait, i.e. after this grid has completed)
  __syncthreads();
  if (cl) cluster_sync_all();  // the leader has read every CTA's partial: they may exit
#ifdef RAAS_DBG_TIMING
  if (threadIdx.x == 0 && blockIdx.x < 256) g_raas_tl[p.dbg_slot & 7][blockIdx.x][3] = dbg_gtimer();
#endif
  if (threadIdx.x == 0) {
    const int done = atomicAdd(p.sched + 1, 1);
    if (done == (int)gridDim.x - 1) {
      p.sched[0] = 0;
      p.sched[1] = 0;
    }
  }
}

}  // namespace raas
