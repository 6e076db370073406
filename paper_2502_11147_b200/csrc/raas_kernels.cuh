// raas_kernels.cuh — the libraas device code (sm_100a).
//
//   raas_decode_kernel   one launch = one decode step of one layer for every unit:
//                        slot selection (a1), in-place K/V write (a2), split-K flash-decode over
//                        the L slots (a3), page-max logits (a4), and — in the warp that finishes
//                        a unit's last split — LSE combine (a5), threshold + stamp (a6) and the
//                        next-victim argmin / cursor advance (a7).   SURVEY.md §8(a).
//   raas_prefill_copy / raas_meta_init / raas_refresh   prompt pages + metadata.
//
// Paper: page-based RaaS, §3.3 :143-151, App. B :358-398; readings D1-D20 in DESIGN.md.
//
// Data layout (one handle = one layer, `units` = batch * n_kv_heads):
//   KV store     [units][C][2][16][D] bf16: a page is its 16 K rows followed by its 16 V rows,
//                16*D*4 contiguous bytes moved by ONE bulk copy; inside a token row the 16-byte
//                chunk c is stored at chunk c ^ (row & 7), so the copy lands in shared memory
//                bank-conflict-free for ldmatrix)
//   ts, start, cnt [units][C] int32; npin[units]; plan[units] int4 = {slot, off | evict<<16,
//   used_eff, t} describing the NEXT step (computed at the end of the previous one).
//   pmax [units][C][g] fp32 (log2-domain page-max logits), part_ml [units][nsplit][g] float2,
//   part_acc [units][nsplit][g][D] fp32 (split-K partials, L2 resident), counter[units].
#pragma once
#include "raas_device.cuh"

namespace raas {

constexpr int PAGE = 16;
constexpr int MAX_GROUP = 8;
constexpr int MAX_SPLITS = 80;    // splits per unit (combine scratch in smem)

struct DecodeParams {
  const __nv_bfloat16* q;      // [units*g][D]
  const __nv_bfloat16* k_new;  // [units][D]
  const __nv_bfloat16* v_new;
  __nv_bfloat16* out;          // [units*g][D]
  __nv_bfloat16* kvstore;      // [units][C][2][16][D], chunk-swizzled rows
  int32_t* ts;
  int32_t* start;
  int32_t* cnt;
  const int32_t* npin;
  int4* plan;
  int32_t* counter;
  int32_t* sched;              // [2]: dynamic tile grab counter, CTA exit counter
  float* pmax;
  float* part_acc;
  float2* part_ml;
  uint32_t* status;
  unsigned long long* stats;  // [4]: stamps, decisions, evictions, unit-steps
  int units, C, nsplit, split_pages, g;
  // metadata entries: Ce = L / ep per unit, ep tokens each (ep = 16: pages, the tiles C = Ce;
  // ep = 1: token-level RaaS of PAPER.md §3.2 (NEXT-3), slot s = row s % 16 of tile s / 16)
  int Ce, ep;
  int pstr;  // bf16 elements per page in the KV store: 2 * 16 * D (+ 64: tokd trailer of the
             // tile's 16 ts and 16 start values, copied with the page in ONE bulk copy)
  // token level, threshold rule, per-head tables: DEFERRED stamping (NEXT-3).
  // The step-t decisions need LSE_t, known only after the step-t pass; they are taken in the
  // step-(t+1) pass, row by row, from the stored q_t and LSE_t (an extra S = K q_t^T on the
  // same tile), together with the victim candidates.  The step-(t+1) pass therefore attends
  // the L resident rows, and the combine removes the victim's row and adds the new token.
  int tokd;
  __nv_bfloat16* q_prev;  // [units][g][D] q of the previous step (tokd)
  float* lse_prev;        // [units][8] its log2-domain LSE per q-head (tokd)
  int4* part_key;         // [units][nsplit] victim candidate per split: {key lo, key hi, slot}
  int score_mode;    // 0 exact page max (D4), 1 Quest representative-key bound (D22)
  int stamp_rule;    // 0 threshold alpha (D2/D3), 1 top-r fraction of pages (D23)
  float top_r;
  int quest_k;       // > 0: Quest-on-prefill hybrid (D24), pages selected per step
  const int32_t* nfull;  // [units] full prompt pages (selectable)
  const int32_t* vmap;   // [units][C] selected prompt pages of this step, ascending
  int table_scope;       // 0 per (request, kv-head) tables; 1 one table per request (D25)
  int n_kv;              // kv-heads per request (units of one request are consecutive)
  int dbg_slot;          // RAAS_DBG_TIMING builds: timeline slot of this launch (0..7)
  int cl;                // 1: cluster schedule -- one (unit, split) tile per CTA, the unit's nsplit
                         // CTAs form a thread-block cluster, the split partials go to the leader
                         // (cluster rank 0) through distributed shared memory, no L2 round trip
  int early;             // 1: the previous kernel of the stream is not this handle's decode step,
                         // so this handle's state may be read before griddepcontrol.wait
  uint32_t* req_x;       // [batch][C] table_scope 1: order-preserving max of the page scores
  int32_t* req_ctr;      // [batch]    table_scope 1: kv-heads of the request combined so far
  float scale_log2;  // softmax_scale * log2(e)
  float log2_alpha;  // log2(alpha); -inf for alpha == 0
};

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- argmin over (ts, start_pos) with page index (D12: ties -> oldest page) ------------
struct Cand {
  unsigned long long key;
  int page;
};
__device__ __forceinline__ unsigned long long cand_key(int ts, int start) {
  return (static_cast<unsigned long long>(static_cast<uint32_t>(ts)) << 32) |
         static_cast<uint32_t>(start);
}
__device__ __forceinline__ void cand_update(Cand& c, unsigned long long key, int page) {
  if (key < c.key) { c.key = key; c.page = page; }
}
// every lane returns the warp-wide minimum (keys are unique: start positions are distinct)
__device__ __forceinline__ int warp_argmin_page(const Cand& c) {
  const unsigned long long m = warp_min_u64(c.key);
  const unsigned ball = __ballot_sync(0xffffffffu, c.key == m && c.page >= 0);
  if (ball == 0) return -1;
  return __shfl_sync(0xffffffffu, c.page, __ffs(ball) - 1);
}

// k-th largest (1 <= k <= number of non-zero keys) of the 64-bit keys key[0..n) held in shared
// memory (zero = not a candidate), by one warp: radix select, 8 bits per pass, with a
// 256-bin shared histogram at `hist` (1 KiB).  Every lane returns the key.
__device__ __forceinline__ unsigned long long warp_kth_largest(uint32_t keys, uint32_t hist,
                                                               int n, int k, int lane) {
  unsigned long long prefix = 0, mask = 0;
  int krem = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(hist + 4 * (lane * 8 + j)), "r"(0) : "memory");
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      unsigned long long key;
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(key) : "r"(keys + 8 * i));
      if (key != 0 && (key & mask) == prefix)
        atomicAdd(reinterpret_cast<int*>(__cvta_shared_to_generic(hist)) + ((key >> shift) & 255), 1);
    }
    __syncwarp();
    int c[8], tot = 0;  // lane l owns digits 255-8l .. 248-8l (descending)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(c[j]) : "r"(hist + 4 * (255 - (lane * 8 + j))));
      tot += c[j];
    }
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int excl = incl - tot;
    const unsigned hit = __ballot_sync(0xffffffffu, excl < krem && incl >= krem);
    const int src = __ffs(hit) - 1;
    int digit = 0, above = 0, csel = 0;
    if (lane == src) {
      int run = excl;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (run + c[j] >= krem) { digit = 255 - (lane * 8 + j); above = run; csel = c[j]; break; }
        run += c[j];
      }
    }
    digit = __shfl_sync(0xffffffffu, digit, src);
    above = __shfl_sync(0xffffffffu, above, src);
    csel = __shfl_sync(0xffffffffu, csel, src);
    krem -= above;
    prefix |= static_cast<unsigned long long>(digit) << shift;
    mask |= 255ull << shift;
    __syncwarp();
    if (csel == 1 && shift > 0) {  // one key left in the selected bucket: it is the k-th largest
      unsigned long long hitkey = 0;
      for (int i = lane; i < n; i += 32) {
        unsigned long long key;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(key) : "r"(keys + 8 * i));
        if (key != 0 && (key & mask) == prefix) hitkey = key;
      }
      const unsigned who = __ballot_sync(0xffffffffu, hitkey != 0);
      return __shfl_sync(0xffffffffu, hitkey, __ffs(who) - 1);
    }
  }
  return prefix;
}

// sortable 64-bit ranking key: larger float first, then smaller tie index; never 0
__device__ __forceinline__ unsigned long long rank_key(float x, uint32_t tie) {
  const uint32_t b = __float_as_uint(x);
  const uint32_t sx = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return (static_cast<unsigned long long>(sx) << 32) | (0xffffffffu - tie);
}

// plan for the step after one that left `cnt_slot` tokens in entry `slot` at time t (entries
// of ep tokens, Ce of them; used_eff in use): keep filling, open the next entry, or evict
__device__ __forceinline__ int4 next_plan(int slot, int cnt_slot, int used_eff, int C, int t,
                                          int victim, uint32_t* status, int ep) {
  if (cnt_slot < ep) return make_int4(slot, cnt_slot, used_eff, t + 1);
  if (used_eff < C) return make_int4(used_eff, 0, used_eff + 1, t + 1);
  if (victim < 0) { atomicOr(status, 1u); victim = slot; }
  return make_int4(victim, 1 << 16, used_eff, t + 1);
}

}  // namespace raas

#include "raas_decode.cuh"  // the fused decode-step kernel

namespace raas {

// ===========================================================================================
// Prefill: copy the prompt's K/V rows into pages 0..Pp-1 (16-byte vectors).
// ===========================================================================================
template <int D>
__global__ void raas_prefill_copy(const __nv_bfloat16* __restrict__ k,
                                  const __nv_bfloat16* __restrict__ v, __nv_bfloat16* kvstore,
                                  const int32_t* __restrict__ plen, int units, int n_kv_heads,
                                  int P_max, int C, int pstr) {
  // k, v: [units][P_max][D]; unit u = (b, kv-head) copies its request's first plen[b] tokens
  constexpr int NCH = D / 8;
  const size_t total = (size_t)units * P_max * NCH;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % NCH);
    const size_t src = i / NCH;  // unit * P_max + j
    const int j = (int)(src % P_max);
    const size_t u = src / P_max;
    if (j >= plen[u / n_kv_heads]) continue;
    const int r = j % PAGE;
    const size_t dst = (u * C + j / PAGE) * pstr + (size_t)r * D + (ch ^ (r & 7)) * 8;
    *reinterpret_cast<uint4*>(kvstore + dst) =
        __ldg(reinterpret_cast<const uint4*>(k + src * D) + ch);
    *reinterpret_cast<uint4*>(kvstore + dst + PAGE * D) =
        __ldg(reinterpret_cast<const uint4*>(v + src * D) + ch);
  }
}

// metadata after prefill: unit u's pages < Pp(u) pinned and full (the last may be partial),
// t = P(u), with P(u) = plen[u / n_kv_heads] (variable prompt lengths, NEXT-2)
__global__ void raas_meta_init(int32_t* ts, int32_t* start, int32_t* cnt, int32_t* npin,
                               int32_t* nfull, int4* plan, const int32_t* __restrict__ plen,
                               int units, int n_kv_heads, int C, int ep) {
  // C entries of ep tokens per unit (ep = 16 pages, ep = 1 token slots)
  const size_t total = (size_t)units * C;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int pg = (int)(i % C);
    const size_t u = i / C;
    const int P = plen[u / n_kv_heads];
    const int Pp = (P + ep - 1) / ep;
    ts[i] = 0;
    start[i] = pg < Pp ? pg * ep + 1 : 0;
    cnt[i] = pg < Pp ? min(ep, P - pg * ep) : 0;
    if (pg == 0) {
      npin[u] = Pp;
      nfull[u] = P / ep;  // full prompt pages: selectable by the hybrid mode (D24)
      plan[u] = make_int4(0, 0, 0, P + 1);  // .w = t + 1; the rest derived by raas_refresh
    }
  }
}

// Derive the next-step plan of every unit from its metadata (after prefill / set_state).
// One warp per unit.  Reads t from plan[u].w - 1.
__global__ void raas_refresh(const int32_t* ts, const int32_t* start, const int32_t* cnt,
                             const int32_t* npin, int4* plan, int32_t* counter, uint32_t* status,
                             int units, int C, int ep, int tokd) {
  const int unit = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (unit >= units) return;
  const int t = plan[unit].w - 1;
  const int np = npin[unit];
  int used = 0;
  unsigned long long cur_key = 0;  // (start << 32 | page+1), max -> current page
  Cand best{~0ull, -1};
  for (int pg = lane; pg < C; pg += 32) {
    const size_t ix = (size_t)unit * C + pg;
    if (cnt[ix] > 0) {
      ++used;
      const unsigned long long k =
          (static_cast<unsigned long long>(static_cast<uint32_t>(start[ix])) << 32) | (pg + 1);
      cur_key = k > cur_key ? k : cur_key;
      if (pg >= np) cand_update(best, cand_key(ts[ix], start[ix]), pg);
    }
  }
  used = warp_sum_i(used);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, cur_key, o);
    cur_key = w > cur_key ? w : cur_key;
  }
  const int victim = warp_argmin_page(best);
  if (lane == 0) {
    int4 pl;
    if (tokd) {
      // deferred token-level plan: {fill slot or -1, pending decisions, used rows, t + 1}
      pl = make_int4(used < C ? used : -1, 0, used, t + 1);
    } else if (cur_key == 0) {
      pl = make_int4(0, 0, 1, t + 1);  // nothing resident yet (P == 0): open page 0
    } else {
      const int cur = (int)(cur_key & 0xffffffffu) - 1;
      pl = next_plan(cur, cnt[(size_t)unit * C + cur], used, C, t, victim, status, ep);
    }
    plan[unit] = pl;
    counter[unit] = 0;
  }
}

// Deferred token-level stamping (tokd): apply the decisions still pending from the last step
// (before a state readout).  One block per unit; x_j = max_h (scale q_h . k_j - LSE_h) in the
// log2 domain from the stored q and LSE, stamp iff x_j > log2(alpha) (strict, D3), unpinned rows.
template <int D>
__global__ void raas_tok_flush(__nv_bfloat16* kvstore,
                               const __nv_bfloat16* __restrict__ q_prev,
                               const float* __restrict__ lse_prev, int32_t* ts,
                               const int32_t* __restrict__ npin, int4* plan,
                               unsigned long long* stats, int C, int g, float scale_log2,
                               float log2_alpha, int pstr) {
  const int unit = blockIdx.x;
  const int4 pl = plan[unit];
  if (pl.y == 0) return;  // nothing pending
  const int used = pl.z, tm1 = pl.w - 1, np = npin[unit];
  __shared__ float qs[MAX_GROUP][D];
  __shared__ int cnt_s[2];
  for (int i = threadIdx.x; i < g * D; i += blockDim.x)
    qs[i / D][i % D] = __bfloat162float(q_prev[(size_t)unit * g * D + i]);
  if (threadIdx.x < 2) cnt_s[threadIdx.x] = 0;
  __syncthreads();
  int n_dec = 0, n_stamp = 0;
  for (int j = np + threadIdx.x; j < used; j += blockDim.x) {
    const int tile = j / PAGE, r = j % PAGE;
    const __nv_bfloat16* krow = kvstore + (size_t)(unit * (C / PAGE) + tile) * pstr + (size_t)r * D;
    float x = -INFINITY;
    for (int h = 0; h < g; ++h) {
      float acc = 0.f;
      for (int c = 0; c < D; ++c)  // chunk c / 8 of the row is stored at chunk (c / 8) ^ (r & 7)
        acc += qs[h][c] * __bfloat162float(krow[(((c >> 3) ^ (r & 7)) << 3) | (c & 7)]);
      x = fmaxf(x, acc * scale_log2 - lse_prev[unit * 8 + h]);
    }
    ++n_dec;
    if (x > log2_alpha) {
      ts[(size_t)unit * C + j] = tm1;
      reinterpret_cast<int32_t*>(kvstore + (size_t)(unit * (C / PAGE) + tile) * pstr + 2 * PAGE * D)[r] = tm1;
      ++n_stamp;
    }
  }
  atomicAdd(&cnt_s[0], n_dec);
  atomicAdd(&cnt_s[1], n_stamp);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(stats + 0, (unsigned long long)cnt_s[1]);
    atomicAdd(stats + 1, (unsigned long long)cnt_s[0]);
    plan[unit].y = 0;
  }
}

// tokd: copy the ts / start arrays into the pages' trailers (after prefill and set_state)
__global__ void raas_tok_trailer_sync(__nv_bfloat16* kvstore, const int32_t* __restrict__ ts,
                                      const int32_t* __restrict__ start, size_t tiles, int pstr) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tiles * 32;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t tl = i / 32;
    const int k = (int)(i % 32);
    const size_t e = tl * PAGE + (k & (PAGE - 1));  // entry (token slot) of this trailer word
    reinterpret_cast<int32_t*>(kvstore + tl * pstr + (pstr - 64))[k] = k < PAGE ? ts[e] : start[e];
  }
}

// ------------------------------------------------------------------------------------------
// Quest-on-prefill + RaaS-on-decode hybrid (SURVEY NEXT-4; PAPER.md :173/:183, :237; D24)
// ------------------------------------------------------------------------------------------
// Quest score mode (score_mode 1, NEXT-1): every page's per-channel min / max key rows live in
// the page's HBM trailer (after its 16 V rows), maintained by the decode kernel on every write.
// This kernel (re)builds them from the store over each page's valid rows [0, cnt) -- after
// prefill and raas_set_state.  Empty pages get +inf / -inf (never read: they are not resident).
template <int D>
__global__ void raas_qtrailer_kernel(__nv_bfloat16* kvstore, const int32_t* __restrict__ cnt,
                                     int units, int C, int pstr) {
  constexpr int NCH = D / 8;
  const size_t total = (size_t)units * C * NCH;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % NCH);
    const size_t pu = i / NCH;
    const int n = cnt[pu];
    __nv_bfloat16* kp = kvstore + pu * pstr;
    uint32_t mn[4] = {0x7f807f80u, 0x7f807f80u, 0x7f807f80u, 0x7f807f80u};
    uint32_t mx[4] = {0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u};
    for (int r = 0; r < n; ++r) {
      const uint4 w = *(reinterpret_cast<const uint4*>(kp + r * D) + (ch ^ (r & 7)));
      const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        asm("min.bf16x2 %0, %0, %1;" : "+r"(mn[e]) : "r"(wv[e]));
        asm("max.bf16x2 %0, %0, %1;" : "+r"(mx[e]) : "r"(wv[e]));
      }
    }
    *reinterpret_cast<uint4*>(kp + 2 * PAGE * D + ch * 8) = make_uint4(mn[0], mn[1], mn[2], mn[3]);
    *reinterpret_cast<uint4*>(kp + 2 * PAGE * D + D + ch * 8) = make_uint4(mx[0], mx[1], mx[2], mx[3]);
  }
}

// Representative keys of the full prompt pages: per channel min and max over the 16 keys
// (exact in bf16), repkey [units][C][2][D].
template <int D>
__global__ void raas_repkey_kernel(const __nv_bfloat16* __restrict__ kvstore,
                                   __nv_bfloat16* repkey, const int32_t* __restrict__ nfull,
                                   int units, int C, int pstr) {
  constexpr int NCH = D / 8;
  const size_t total = (size_t)units * C * NCH;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % NCH);
    const size_t pu = i / NCH;
    const int pg = (int)(pu % C);
    const size_t u = pu / C;
    if (pg >= nfull[u]) continue;
    const __nv_bfloat16* kp = kvstore + pu * pstr;
    uint32_t mn[4] = {0x7f807f80u, 0x7f807f80u, 0x7f807f80u, 0x7f807f80u};
    uint32_t mx[4] = {0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u};
#pragma unroll
    for (int r = 0; r < PAGE; ++r) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(kp + r * D) + (ch ^ (r & 7)));
      const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        asm("min.bf16x2 %0, %0, %1;" : "+r"(mn[e]) : "r"(wv[e]));
        asm("max.bf16x2 %0, %0, %1;" : "+r"(mx[e]) : "r"(wv[e]));
      }
    }
    *reinterpret_cast<uint4*>(repkey + (pu * 2 + 0) * D + ch * 8) = make_uint4(mn[0], mn[1], mn[2], mn[3]);
    *reinterpret_cast<uint4*>(repkey + (pu * 2 + 1) * D + ch * 8) = make_uint4(mx[0], mx[1], mx[2], mx[3]);
  }
}

// Per step: Quest bound of every full prompt page (max over the group's heads of
// sum_c max(q_c min_c, q_c max_c)) and the top-K pages by (bound desc, page asc) ->
// vmap[u][0..K) in ascending page order.  One 256-thread block per unit, PDL-chained in front
// of the decode kernel.  The representative keys are static after prefill, so the first 2 * 32
// pages' min/max rows are loaded BEFORE griddepcontrol.wait;
// only q waits.  8 lanes per page (D/8 channels each), 32 pages per pass.  (128-thread blocks
// that fit beside a resident decode CTA were measured slower: 2.81 vs 2.56 ms per step.)  Selection by rank:
// page p is selected iff fewer than K keys beat its key (keys are unique), then warp 0 writes
// the selected pages in ascending order.  Shared memory: g*D*4 (q) + 8*C (keys) + C (flags).
constexpr int QSEL_THREADS = 256;
template <int D>
__global__ void __launch_bounds__(QSEL_THREADS) raas_qselect_kernel(const __nv_bfloat16* __restrict__ q,
                                    const __nv_bfloat16* __restrict__ repkey,
                                    const int32_t* __restrict__ nfull, int32_t* vmap, int units,
                                    int C, int g, int K) {
  extern __shared__ uint8_t qs_smem[];
  constexpr int CH = D / 8;  // channels per lane
  constexpr int PPASS = QSEL_THREADS / 8;  // pages per pass (8 lanes per page)
  const int u = blockIdx.x;
  const int nf = nfull[u];   // written by prefill / set_state only
  const int sub = threadIdx.x >> 3, cl = threadIdx.x & 7;
  // min / max of this lane's channels {32 v + 4 cl + e} (bank-conflict-free q reads) of its
  // first two pages, as bf16x2 words, loaded before the dependency wait
  constexpr int NV = CH / 4;
  uint32_t mnw[2][CH / 2], mxw[2][CH / 2];
  auto load_page = [&](int pg, int slot) {
    const size_t pu = (size_t)u * C + (pg < C ? pg : C - 1);  // independent of nf (no wait)
    const __nv_bfloat16* mnp = repkey + (pu * 2 + 0) * D + 4 * cl;
    const __nv_bfloat16* mxp = repkey + (pu * 2 + 1) * D + 4 * cl;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const uint2 a = __ldg(reinterpret_cast<const uint2*>(mnp + 32 * v));
      const uint2 b = __ldg(reinterpret_cast<const uint2*>(mxp + 32 * v));
      mnw[slot][2 * v] = a.x; mnw[slot][2 * v + 1] = a.y;
      mxw[slot][2 * v] = b.x; mxw[slot][2 * v + 1] = b.y;
    }
  };
  load_page(sub, 0);
  load_page(sub + PPASS, 1);
  const bool active = nf > K;  // block-uniform: otherwise every prompt page is attended
  pdl_wait();  // q of this step is produced by earlier work in the stream
  pdl_launch_dependents();
  if (!active) return;
  float* qf = reinterpret_cast<float*>(qs_smem);
  const uint32_t keys = smem_u32(qs_smem) + g * D * 4;
  uint8_t* selb = qs_smem + g * D * 4 + 8 * C;
  for (int i = threadIdx.x; i < g * D; i += blockDim.x)
    qf[i] = __bfloat162float(q[(size_t)u * g * D + i]);
  __syncthreads();
  // bound of page pg from min / max words held in registers (compile-time indexed)
  auto do_page = [&](const uint32_t (&mn)[CH / 2], const uint32_t (&mx)[CH / 2], int pg) {
    float sc = -INFINITY;
#pragma unroll
    for (int h = 0; h < MAX_GROUP; ++h) {
      if (h < g) {
        const float4* qh = reinterpret_cast<const float4*>(qf + h * D + 4 * cl);
        float U = 0.f;
#pragma unroll
        for (int c4 = 0; c4 < NV; ++c4) {
          const float4 qv = qh[8 * c4];  // channels 32 c4 + 4 cl + (0..3)
          const float qa[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = 4 * c4 + e;
            const uint32_t sh = (c & 1) ? 0u : 16u;
            const float a = __uint_as_float((mn[c >> 1] << sh) & 0xffff0000u);
            const float b = __uint_as_float((mx[c >> 1] << sh) & 0xffff0000u);
            U += fmaxf(qa[e] * a, qa[e] * b);
          }
        }
        U += __shfl_xor_sync(0xffffffffu, U, 1);
        U += __shfl_xor_sync(0xffffffffu, U, 2);
        U += __shfl_xor_sync(0xffffffffu, U, 4);
        sc = fmaxf(sc, U);
      }
    }
    if (pg < nf && cl == 0) {
      const unsigned long long key = rank_key(sc, (uint32_t)pg);
      asm volatile("st.shared.u64 [%0], %1;" ::"r"(keys + 8 * pg), "l"(key) : "memory");
    }
  };
  do_page(mnw[0], mxw[0], sub);
  if (nf > PPASS) do_page(mnw[1], mxw[1], sub + PPASS);
  for (int p0 = 2 * PPASS; p0 < nf; p0 += PPASS) {  // pages beyond the prefetched ones
    load_page(p0 + sub, 0);
    do_page(mnw[0], mxw[0], p0 + sub);
  }
  __syncthreads();
  // rank of every page's key among the nf keys; selected iff fewer than K are larger
  for (int pg = threadIdx.x; pg < nf; pg += blockDim.x) {
    unsigned long long kp;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(kp) : "r"(keys + 8 * pg));
    int above = 0;
#pragma unroll 8
    for (int j = 0; j < nf; ++j) {
      unsigned long long kj;
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(kj) : "r"(keys + 8 * j));
      above += kj > kp ? 1 : 0;
    }
    selb[pg] = above < K ? 1 : 0;
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int base = 0;
  for (int c0 = 0; c0 < nf; c0 += 32) {  // ascending compaction of the selected pages
    const int pg = c0 + lane;
    const bool sel = pg < nf && selb[pg];
    const unsigned b = __ballot_sync(0xffffffffu, sel);
    if (sel) vmap[(size_t)u * C + base + __popc(b & ((1u << lane) - 1))] = pg;
    base += __popc(b);
  }
}

// raas_decode_step_host with pinned (mapped) host buffers: one step's q / k_new / v_new are
// read from host memory over PCIe by the SMs (zero-copy) and stored into the arena's staging
// area.  The host reads are issued BEFORE griddepcontrol.wait (the host buffers are complete
// when the call is made), so they overlap the previous kernel of the stream; the stores wait
// for it (the staging area may still be read by this handle's previous step).  The decode
// kernel is triggered at once, so its prologue overlaps the previous kernel's tail too.  128-thread
// blocks with a small register budget fit beside a resident decode CTA.  Counts in 16 B
// vectors; element i of the concatenation [q | k | v].
constexpr int INGEST_THREADS = 128, INGEST_PER = 4;
__global__ void __launch_bounds__(INGEST_THREADS) raas_ingest_kernel(
    const uint4* __restrict__ q_h, const uint4* __restrict__ k_h, const uint4* __restrict__ v_h,
    uint4* __restrict__ q_d, uint4* __restrict__ k_d, uint4* __restrict__ v_d, int nq, int nkv,
    int store_early) {
  const int total = nq + 2 * nkv;
  const int nth = gridDim.x * INGEST_THREADS;
  const int tid = blockIdx.x * INGEST_THREADS + threadIdx.x;
  auto ld = [&](int i) {
    return i < nq ? ld_sys_v4(q_h + i) : i < nq + nkv ? ld_sys_v4(k_h + (i - nq)) : ld_sys_v4(v_h + (i - nq - nkv));
  };
  auto st = [&](int i, uint4 x) {
    if (i < nq) q_d[i] = x;
    else if (i < nq + nkv) k_d[i - nq] = x;
    else v_d[i - nq - nkv] = x;
  };
  // the decode step may start (its state reads and first page copies) at once: it reads q /
  // k_new / v_new only after its own griddepcontrol.wait, i.e. after this grid has completed,
  // and this grid completes only after the previous kernel of the stream (our wait below).
  // store_early (the previous decode launch on the stream is another handle's, so nothing still
  // running reads this handle's staging buffers): the whole copy runs before the wait, which
  // then only keeps the chain ordered; otherwise the stores wait (a handle stepped twice in a
  // row: its previous decode may still read q from the staging buffer)
  pdl_launch_dependents();
  uint4 r[INGEST_PER];
#pragma unroll
  for (int j = 0; j < INGEST_PER; ++j) {
    const int i = tid + j * nth;
    if (i < total) r[j] = ld(i);
  }
  if (!store_early) pdl_wait();
#pragma unroll
  for (int j = 0; j < INGEST_PER; ++j) {
    const int i = tid + j * nth;
    if (i < total) st(i, r[j]);
  }
  for (int i0 = tid + INGEST_PER * nth; i0 < total; i0 += INGEST_PER * nth) {  // large batches
#pragma unroll
    for (int j = 0; j < INGEST_PER; ++j) {
      const int i = i0 + j * nth;
      if (i < total) r[j] = ld(i);
    }
#pragma unroll
    for (int j = 0; j < INGEST_PER; ++j) {
      const int i = i0 + j * nth;
      if (i < total) st(i, r[j]);
    }
  }
  if (store_early) pdl_wait();  // completes only after the previous kernel: the chain holds
}

}  // namespace raas
