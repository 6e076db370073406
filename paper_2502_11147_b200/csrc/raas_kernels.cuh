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
//   K, V store   [units][C][16][D] bf16           (a page = 16*D*2 contiguous bytes)
//   ts, start, cnt [units][C] int32; npin[units]; plan[units] int4 = {slot, off | evict<<16,
//   used_eff, t} describing the NEXT step (computed at the end of the previous one).
//   pmax [units][C][g] fp32 (log2-domain page-max logits), part_ml [units][nsplit][g] float2,
//   part_acc [units][nsplit][g][D] fp32 (split-K partials, L2 resident), counter[units].
#pragma once
#include "raas_device.cuh"

namespace raas {

constexpr int PAGE = 16;
constexpr int MAX_GROUP = 8;
constexpr int MAX_SPLITS = 128;   // splits per unit (combine: 4 per lane)

struct DecodeParams {
  const __nv_bfloat16* q;      // [units*g][D]
  const __nv_bfloat16* k_new;  // [units][D]
  const __nv_bfloat16* v_new;
  __nv_bfloat16* out;          // [units*g][D]
  __nv_bfloat16* kstore;
  __nv_bfloat16* vstore;
  int32_t* ts;
  int32_t* start;
  int32_t* cnt;
  const int32_t* npin;
  int4* plan;
  int32_t* counter;
  float* pmax;
  float* part_acc;
  float2* part_ml;
  uint32_t* status;
  unsigned long long* stats;  // [4]: stamps, decisions, evictions, unit-steps
  int units, C, nsplit, split_pages, g;
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

// plan for the step after one that wrote `off_written` (0-based) into `slot` at time t
__device__ __forceinline__ int4 next_plan(int slot, int cnt_slot, int used_eff, int C, int t,
                                          int victim, uint32_t* status) {
  if (cnt_slot < PAGE) return make_int4(slot, cnt_slot, used_eff, t + 1);
  if (used_eff < C) return make_int4(used_eff, 0, used_eff + 1, t + 1);
  if (victim < 0) { atomicOr(status, 1u); victim = slot; }
  return make_int4(victim, 1 << 16, used_eff, t + 1);
}

// ===========================================================================================
// Decode step.  Persistent; every WARP is an independent flash-decode worker that owns whole
// split tiles (unit, split) in the static order gw, gw + TW, ...  Its lane 0 keeps STAGES
// pages (K 16xD + V 16xD, bf16, 128B-swizzled by TMA) in flight through a private mbarrier
// ring; QK^T and PV run on bf16 mma.sync m16n8k16 with the 16 tokens of a page as M and the
// (<= 8) q-heads of the GQA group as N; softmax state in fp32 registers.
// ===========================================================================================
template <int D, int NW, int STAGES>
__global__ void __launch_bounds__(NW * 32)
    raas_decode_kernel(const __grid_constant__ DecodeParams p,
                       const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV) {
  static_assert(D == 64 || D == 128, "head_dim");
  constexpr int KS = D / 16;                 // k-steps of QK^T == m-tiles of PV
  constexpr int HALVES = D / 64;             // 128-byte TMA boxes per row
  constexpr int TILE = PAGE * D * 2;         // bytes of one K (or V) page
  constexpr int STAGE = 2 * TILE;
  constexpr int DPL = D / 32;                // output dims per lane in the combine

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // 128B swizzle atoms need 1024B alignment
  uint8_t* sm = smem_raw + (base - raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t wtiles = base + warp * STAGES * STAGE;
  const uint32_t wbars = base + NW * STAGES * STAGE + warp * STAGES * 8;
  int4* winfo = reinterpret_cast<int4*>(sm + NW * STAGES * STAGE + NW * STAGES * 8) +
                warp * STAGES * 2;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(wbars + 8 * s, 1);
    fence_mbar_init();
  }
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  __syncwarp();
  // PDL: everything above overlapped the previous kernel's tail; state reads start here.
  pdl_wait();
  pdl_launch_dependents();

  const int C = p.C, SP = p.split_pages, g = p.g;
  const int TW = gridDim.x * NW;
  const int n_tiles = p.units * p.nsplit;
  const uint64_t pol = l2_evict_first_policy();

  // ---------------- load iterator (warp-uniform) ----------------
  int ld_tile = blockIdx.x * NW + warp - TW;
  int ld_p = 0, ld_pend = 0, ld_p0 = 0, ld_unit = 0, ld_split = 0, ld_nse = 0, ld_cnt = 0;
  int4 ld_plan = make_int4(0, 0, 0, 0);
  bool ld_done = false;

  auto advance = [&]() {
    while (ld_p >= ld_pend) {
      ld_tile += TW;
      if (ld_tile >= n_tiles) { ld_done = true; return; }
      ld_unit = ld_tile / p.nsplit;
      ld_split = ld_tile - ld_unit * p.nsplit;
      ld_plan = p.plan[ld_unit];
      const int used_eff = ld_plan.z;
      ld_p0 = ld_split * SP;
      ld_p = ld_p0;
      ld_pend = min(ld_p0 + SP, used_eff);
      ld_nse = (used_eff + SP - 1) / SP;
      if (ld_p < ld_pend)
        ld_cnt = (lane < ld_pend - ld_p0) ? p.cnt[ld_unit * C + ld_p0 + lane] : 0;
    }
  };

  auto issue = [&](int s) {
    const int page = ld_p;
    const int slot = ld_plan.x, off = ld_plan.y & 0xffff;
    const int c = __shfl_sync(0xffffffffu, ld_cnt, page - ld_p0);
    const bool is_slot = (page == slot);
    if (lane == 0) {
      winfo[2 * s] = make_int4(ld_unit, page, is_slot ? off + 1 : c, is_slot ? off : -1);
      winfo[2 * s + 1] =
          make_int4(ld_split, page + 1 == ld_pend ? 1 : 0, ld_nse, page == ld_p0 ? 1 : 0);
      const uint32_t bar = wbars + 8 * s;
      mbar_arrive_expect_tx(bar, STAGE);
      const int32_t y = (ld_unit * C + page) * PAGE;
      const uint32_t dk = wtiles + s * STAGE, dv = dk + TILE;
#pragma unroll
      for (int hf = 0; hf < HALVES; ++hf) {
        tma_load_2d(dk + hf * 2048, &tmK, hf * 64, y, bar, pol);
        tma_load_2d(dv + hf * 2048, &tmV, hf * 64, y, bar, pol);
      }
    }
    ++ld_p;
  };

  // ---------------- compute state ----------------
  const int r = lane >> 2, qd = lane & 3;          // C-fragment row (token) / column pair (head)
  const int mi = lane >> 3, ri = lane & 7;         // ldmatrix matrix / row supplied by this lane
  float acc[KS][4];
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  uint32_t qb[KS][2];

  int issued = 0, consumed = 0;
  advance();
  while (!ld_done && issued < STAGES) {
    issue(issued);
    ++issued;
    advance();
  }

  while (consumed < issued) {
    const int s = consumed % STAGES;
    mbar_wait(wbars + 8 * s, (consumed / STAGES) & 1);
    const int4 i0 = winfo[2 * s], i1 = winfo[2 * s + 1];
    const int unit = i0.x, page = i0.y, cnt = i0.z, patch = i0.w;
    const uint32_t kb = wtiles + s * STAGE, vb = kb + TILE;

    if (i1.w) {  // first page of a tile: fresh softmax state, this unit's q fragments
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.f;
      const uint32_t* qrow =
          reinterpret_cast<const uint32_t*>(p.q + (size_t)(unit * g + r) * D) + qd;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        qb[ks][0] = r < g ? __ldg(qrow + ks * 8) : 0u;      // d = 16ks + 2qd, +1
        qb[ks][1] = r < g ? __ldg(qrow + ks * 8 + 4) : 0u;  // d = 16ks + 8 + 2qd, +1
      }
    }

    if (patch >= 0) {  // a2: the new token's K/V go to row `patch` of this page (smem + HBM)
      constexpr int NCH = D / 8;  // 16-byte chunks per row
      if (lane < 2 * NCH) {
        const bool isv = lane >= NCH;
        const int ch = isv ? lane - NCH : lane;
        const uint4 val = __ldg(reinterpret_cast<const uint4*>(
                                    (isv ? p.v_new : p.k_new) + (size_t)unit * D) + ch);
        const uint32_t sa = (isv ? vb : kb) + (ch >> 3) * 2048 + patch * 128 +
                            (((ch & 7) ^ (patch & 7)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(sa), "r"(val.x), "r"(val.y),
                     "r"(val.z), "r"(val.w)
                     : "memory");
        __nv_bfloat16* g_dst = (isv ? p.vstore : p.kstore) +
                               ((size_t)(unit * C + page) * PAGE + patch) * D + ch * 8;
        *reinterpret_cast<uint4*>(g_dst) = val;
        fence_proxy_async_smem();
      }
      __syncwarp();
    }

    // ---- a3/a4: S^T = K_page . Q^T  (M = 16 tokens, N = 8 heads, K = D) ----
    float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
    {
      const uint32_t krow = kb + (ri + 8 * (mi & 1)) * 128;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        uint32_t a[4];
        const int chunk = 2 * (ks & 3) + (mi >> 1);
        ldsm_x4(krow + (ks >> 2) * 2048 + ((chunk ^ ri) << 4), a);
        if (ks & 1) mma_bf16_16816(c1, a, qb[ks][0], qb[ks][1]);
        else        mma_bf16_16816(c0, a, qb[ks][0], qb[ks][1]);
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
    if (lane < 4) {  // a4: page-max logit per head ("a single attention score per page", :147)
      float* pmx = p.pmax + (size_t)(unit * C + page) * g;
      if (2 * qd < g) pmx[2 * qd] = pm0;
      if (2 * qd + 1 < g) pmx[2 * qd + 1] = pm1;
    }
    const float mn0 = fmaxf(m0, pm0), mn1 = fmaxf(m1, pm1);
    const float cr0 = fast_exp2(m0 - mn0), cr1 = fast_exp2(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    const float p0 = fast_exp2(s0 - mn0), p1 = fast_exp2(s1 - mn1);
    const float p2 = fast_exp2(s2 - mn0), p3 = fast_exp2(s3 - mn1);
    l0 = l0 * cr0 + (p0 + p2);
    l1 = l1 * cr1 + (p1 + p3);
#pragma unroll
    for (int mt = 0; mt < KS; ++mt) {
      acc[mt][0] *= cr0;
      acc[mt][1] *= cr1;
      acc[mt][2] *= cr0;
      acc[mt][3] *= cr1;
    }
    // P^T as the B operand of O^T = V^T P^T: transpose the two 8x8 bf16 blocks in registers
    const uint32_t b0 = movmatrix_t(pack_bf16x2(p0, p1));
    const uint32_t b1 = movmatrix_t(pack_bf16x2(p2, p3));
    {
      const uint32_t vrow = vb + (ri + 8 * (mi >> 1)) * 128;
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        uint32_t a[4];
        const int chunk = 2 * (mt & 3) + (mi & 1);
        ldsm_x4_t(vrow + (mt >> 2) * 2048 + ((chunk ^ ri) << 4), a);
        mma_bf16_16816(acc[mt], a, b0, b1);
      }
    }
    __syncwarp();
    ++consumed;
    if (!ld_done) {  // refill the stage just drained
      issue(s);
      ++issued;
      advance();
    }

    if (i1.y) {  // last page of the tile: publish the split-K partial
      const int split = i1.x, nse = i1.z;
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
      }
      const int pbase = (unit * p.nsplit + split) * g;
      if (lane < 4) {
        if (2 * qd < g) p.part_ml[pbase + 2 * qd] = make_float2(m0, l0);
        if (2 * qd + 1 < g) p.part_ml[pbase + 2 * qd + 1] = make_float2(m1, l1);
      }
      float* pa0 = p.part_acc + (size_t)(pbase + 2 * qd) * D + r;
      float* pa1 = pa0 + D;
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        if (2 * qd < g) { pa0[16 * mt] = acc[mt][0]; pa0[16 * mt + 8] = acc[mt][2]; }
        if (2 * qd + 1 < g) { pa1[16 * mt] = acc[mt][1]; pa1[16 * mt + 8] = acc[mt][3]; }
      }
      __threadfence();
      __syncwarp();
      int old = 0;
      if (lane == 0) old = atomicAdd(p.counter + unit, 1);
      old = __shfl_sync(0xffffffffu, old, 0);
      if (old == nse - 1) {
        // ===== this warp finished the unit's last split: a5 combine, a6 stamp, a7 evict =====
        __threadfence();
        const int4 pl = __ldcg(p.plan + unit);
        const int slot = pl.x, off = pl.y & 0xffff, evicting = pl.y >> 16;
        const int used_eff = pl.z, t = pl.w;
        const int npin = __ldg(p.npin + unit);
        float lse[MAX_GROUP];
#pragma unroll
        for (int h = 0; h < MAX_GROUP; ++h) {
          lse[h] = 0.f;
          if (h < g) {
            constexpr int SPL = MAX_SPLITS / 32;  // splits per lane
            float ms[SPL], w[SPL], lsum = 0.f, M = -INFINITY;
#pragma unroll
            for (int k = 0; k < SPL; ++k) {
              const int sp = lane + 32 * k;
              const float2 ml = sp < nse ? __ldcg(p.part_ml + (unit * p.nsplit + sp) * g + h)
                                         : make_float2(-INFINITY, 0.f);
              ms[k] = ml.x;
              w[k] = ml.y;  // holds l until the weights are known
              M = fmaxf(M, ml.x);
            }
            M = warp_max(M);
#pragma unroll
            for (int k = 0; k < SPL; ++k) {
              const float l_k = w[k];
              w[k] = lane + 32 * k < nse ? fast_exp2(ms[k] - M) : 0.f;
              lsum += l_k * w[k];
            }
            const float Lh = warp_sum(lsum);
            lse[h] = M + log2f(Lh);  // log2-domain LSE of head h
            const float inv = 1.f / Lh;
            float o[DPL];
#pragma unroll
            for (int i = 0; i < DPL; ++i) o[i] = 0.f;
#pragma unroll
            for (int k = 0; k < SPL; ++k) {
              for (int j = 0; j < 32 && 32 * k + j < nse; ++j) {
                const int sp = 32 * k + j;
                const float ws = __shfl_sync(0xffffffffu, w[k], j);
                const float* src =
                    p.part_acc + (size_t)((unit * p.nsplit + sp) * g + h) * D + lane * DPL;
                if constexpr (DPL == 4) {
                  const float4 v = __ldcg(reinterpret_cast<const float4*>(src));
                  o[0] += ws * v.x; o[1] += ws * v.y; o[2] += ws * v.z; o[3] += ws * v.w;
                } else {
                  const float2 v = __ldcg(reinterpret_cast<const float2*>(src));
                  o[0] += ws * v.x; o[1] += ws * v.y;
                }
              }
            }
            __nv_bfloat16* dst = p.out + (size_t)(unit * g + h) * D + lane * DPL;
            if constexpr (DPL == 4) {
              uint2 pk = make_uint2(pack_bf16x2(o[0] * inv, o[1] * inv),
                                    pack_bf16x2(o[2] * inv, o[3] * inv));
              *reinterpret_cast<uint2*>(dst) = pk;
            } else {
              *reinterpret_cast<uint32_t*>(dst) = pack_bf16x2(o[0] * inv, o[1] * inv);
            }
          }
        }
        // a6: stamp unpinned resident pages whose page-max normalised score exceeds alpha
        //     (strict, log2 domain: max_h M_hp - LSE_h > log2 alpha); a2 metadata of the slot
        Cand best{~0ull, -1};
        int n_stamp = 0, n_dec = 0;
        for (int pg = lane; pg < C; pg += 32) {
          if (pg < used_eff) {
            const size_t ix = (size_t)unit * C + pg;
            int ts_p = __ldcg(p.ts + ix), st_p = __ldcg(p.start + ix);
            const bool is_slot = pg == slot;
            if (is_slot) {
              if (off == 0) { st_p = t; p.start[ix] = t; }
              p.cnt[ix] = off + 1;
            }
            if (pg >= npin) {
              float x = -INFINITY;
              const float* pm = p.pmax + ix * g;
#pragma unroll
              for (int h = 0; h < MAX_GROUP; ++h)
                if (h < g) x = fmaxf(x, __ldcg(pm + h) - lse[h]);
              const bool stamp = x > p.log2_alpha;
              ++n_dec;
              n_stamp += stamp ? 1 : 0;
              if (stamp || is_slot) { ts_p = t; p.ts[ix] = t; }
              cand_update(best, cand_key(ts_p, st_p), pg);
            }
          }
        }
        // a7: next cursor / victim (argmin (ts, start_pos) over unpinned pages, D11/D12)
        const int victim = warp_argmin_page(best);
        n_stamp = warp_sum_i(n_stamp);
        n_dec = warp_sum_i(n_dec);
        if (lane == 0) {
          p.plan[unit] = next_plan(slot, off + 1, used_eff, C, t, victim, p.status);
          p.counter[unit] = 0;
          atomicAdd(p.stats + 0, (unsigned long long)n_stamp);
          atomicAdd(p.stats + 1, (unsigned long long)n_dec);
          if (evicting) atomicAdd(p.stats + 2, 1ull);
          atomicAdd(p.stats + 3, 1ull);
        }
      }
    }
  }
}

// ===========================================================================================
// Prefill: copy the prompt's K/V rows into pages 0..Pp-1 (16-byte vectors).
// ===========================================================================================
template <int D>
__global__ void raas_prefill_copy(const __nv_bfloat16* __restrict__ k,
                                  const __nv_bfloat16* __restrict__ v, __nv_bfloat16* kstore,
                                  __nv_bfloat16* vstore, int units, int P, int C) {
  constexpr int NCH = D / 8;
  const size_t total = (size_t)units * P * NCH;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % NCH);
    const size_t row = i / NCH;  // unit * P + j
    const int j = (int)(row % P);
    const size_t u = row / P;
    const size_t dst = ((u * C + j / PAGE) * PAGE + (j % PAGE)) * D + ch * 8;
    *reinterpret_cast<uint4*>(kstore + dst) =
        __ldg(reinterpret_cast<const uint4*>(k + row * D) + ch);
    *reinterpret_cast<uint4*>(vstore + dst) =
        __ldg(reinterpret_cast<const uint4*>(v + row * D) + ch);
  }
}

// metadata after prefill: pages < Pp pinned and full (the last may be partial), t = P
__global__ void raas_meta_init(int32_t* ts, int32_t* start, int32_t* cnt, int32_t* npin,
                               int4* plan, int units, int C, int P) {
  const int Pp = (P + PAGE - 1) / PAGE;
  const size_t total = (size_t)units * C;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int pg = (int)(i % C);
    ts[i] = 0;
    start[i] = pg < Pp ? pg * PAGE + 1 : 0;
    cnt[i] = pg < Pp ? min(PAGE, P - pg * PAGE) : 0;
    if (pg == 0) {
      const size_t u = i / C;
      npin[u] = Pp;
      plan[u] = make_int4(0, 0, 0, P + 1);  // .w = t + 1; the rest derived by raas_refresh
    }
  }
}

// Derive the next-step plan of every unit from its metadata (after prefill / set_state).
// One warp per unit.  Reads t from plan[u].w - 1.
__global__ void raas_refresh(const int32_t* ts, const int32_t* start, const int32_t* cnt,
                             const int32_t* npin, int4* plan, int32_t* counter, uint32_t* status,
                             int units, int C) {
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
    if (cur_key == 0) {
      pl = make_int4(0, 0, 1, t + 1);  // nothing resident yet (P == 0): open page 0
    } else {
      const int cur = (int)(cur_key & 0xffffffffu) - 1;
      pl = next_plan(cur, cnt[(size_t)unit * C + cur], used, C, t, victim, status);
    }
    plan[unit] = pl;
    counter[unit] = 0;
  }
}

}  // namespace raas
