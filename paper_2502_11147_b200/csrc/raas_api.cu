// raas_api.cu — host side of libraas: config validation, arena carving, TMA descriptors,
// launches.  The C ABI is declared (and documented, with citations) in include/raas.h.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/raas.h"
#include "raas_kernels.cuh"

using raas::DecodeParams;

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

#define RAAS_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(RAAS_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));           \
  } while (0)

constexpr size_t ALIGN = 1024;
size_t up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }

// decode kernel shape (B200): one persistent CTA per SM with a TMA producer
// warp, a merge/combine warp and NC consumer warps sharing a ring of S page stages.
#ifndef RAAS_NC
#define RAAS_NC 8
#endif
#ifndef RAAS_S
#define RAAS_S 16
#endif
constexpr int NC = RAAS_NC;  // consumer (MMA) warps per CTA
constexpr int S = RAAS_S;    // K+V page stages in the ring (8 KiB each at head_dim 128)
template <int D, bool TOKD = false, bool GEN = false>
using Lay = raas::DecodeLayout<D, NC, S, TOKD, GEN>;
// three instantiations: the default method (lean), every option at run time (gen), and the
// deferred token level (tokd)
template <int D, bool TOKD, bool GEN>
constexpr auto decode_kernel() { return raas::raas_decode_kernel<D, NC, S, TOKD, GEN>; }
template <int D>
constexpr auto decode_kernel_cl() { return raas::raas_decode_kernel<D, NC, S, false, false, true>; }
// one option beside the default method compiled in (raas::F_QUEST / F_TOPR / F_TSC / F_HYB)
template <int D, int FM>
constexpr auto decode_kernel_f() { return raas::raas_decode_kernel<D, NC, S, false, false, false, FM>; }
// one-split units of <= 16 pages (L <= 256 at the default split size; the default method): a half-size CTA
// (4 consumers, 8 stages, 114 KB) so that two fit on an SM and the next layer's CTA streams
// beside the current one's tail (profiles/r02_study.md §6, §10)
constexpr int NC2 = 4, S2 = 8;
template <int D>
constexpr auto decode_kernel_half() { return raas::raas_decode_kernel<D, NC2, S2, false, false>; }
template <int D>
using LayHalf = raas::DecodeLayout<D, NC2, S2, false, false>;

struct Layout {
  size_t kvstore, ts, start, cnt, npin, nfull, plen, plan, repkey, vmap, counter, req_x, req_ctr,
      q_prev, lse_prev, part_key, pmax, part_acc, part_ml, status, sched,
      stats, sq, sk, sv, so, total;
};

struct Derived {
  int C, units, g, split_pages, nsplit;
  int Ce, ep;  // metadata entries per unit (L / page) of ep = page tokens; C = L / 16 tiles
  int tokd;    // token level with deferred stamping (page 1, threshold rule, per-head tables)
  int fm;      // exactly one option beside the default method (raas::F_*): its own instantiation
  int gen;     // any option beyond the default method (page 16, exact score, alpha rule,
               // per-kv-head tables, no Quest-on-prefill): the generic kernel instantiation
  int pstr;    // bf16 elements per KV page: 2 * 16 * D, + 64 (ts/start trailer) when tokd,
               // + 2 * D (the Quest mode's per-channel min / max key rows) when score_mode 1
  int qtr;     // score_mode 1 at page 16: min / max rows maintained in the page trailer
};

int derive(const raas_config* c, Derived* d) {
  if (!c) return fail(RAAS_E_INVALID, "null config");
  if (c->L <= 0 || c->page <= 0 || c->n_q_heads <= 0 || c->n_kv_heads <= 0 ||
      c->head_dim <= 0 || c->batch <= 0)
    return fail(RAAS_E_INVALID, "non-positive size in config");
  if (c->L % c->page != 0) return fail(RAAS_E_INVALID, "L %% page != 0");
  if (c->n_q_heads % c->n_kv_heads != 0) return fail(RAAS_E_INVALID, "n_q_heads %% n_kv_heads != 0");
  if (!(c->alpha >= 0.f)) return fail(RAAS_E_INVALID, "alpha must be >= 0");
  if (c->softmax_scale < 0.f) return fail(RAAS_E_INVALID, "softmax_scale must be >= 0");
  if (c->score_mode != 0 && c->score_mode != 1) return fail(RAAS_E_INVALID, "score_mode must be 0 or 1");
  if (c->stamp_rule != 0 && c->stamp_rule != 1) return fail(RAAS_E_INVALID, "stamp_rule must be 0 or 1");
  if (c->stamp_rule == 1 && !(c->top_r >= 0.f && c->top_r <= 1.f))
    return fail(RAAS_E_INVALID, "top_r must be in [0, 1]");
  if (c->page != raas::PAGE && c->page != 1)
    return fail(RAAS_E_UNSUPPORTED, "page must be 16 (pages) or 1 (token-level RaaS)");
  if (c->L % raas::PAGE != 0) return fail(RAAS_E_UNSUPPORTED, "L must be a multiple of 16");
  d->ep = c->page;
  d->Ce = c->L / c->page;
  d->tokd = c->page == 1 && c->stamp_rule == 0 && c->table_scope == 0 && c->score_mode == 0;
  d->qtr = c->score_mode == 1 && c->page == raas::PAGE;
  d->pstr = 2 * raas::PAGE * c->head_dim + (d->tokd ? 64 : 0) + (d->qtr ? 2 * c->head_dim : 0);
  // exactly one option beside the default method (page 16): its own instantiation with the
  // option compiled in (the generic kernel's run-time options cost 5-8 % at config 3)
  const int fm = (c->score_mode == 1 ? raas::F_QUEST : 0) | (c->stamp_rule == 1 ? raas::F_TOPR : 0) |
                 (c->table_scope != 0 ? raas::F_TSC : 0) | (c->quest_prefill_pages > 0 ? raas::F_HYB : 0);
  d->fm = (!d->tokd && c->page == raas::PAGE && (fm & (fm - 1)) == 0) ? fm : 0;
  if (const char* e = std::getenv("RAAS_GENERIC"))  // tests: the generic kernel for every option
    if (std::atoi(e) != 0) d->fm = 0;
  d->gen = !d->tokd && d->fm == 0 &&
           (c->page != raas::PAGE || c->score_mode != 0 || c->stamp_rule != 0 ||
            c->table_scope != 0 || c->quest_prefill_pages > 0);
  if (c->page == 1 && c->score_mode != 0)
    return fail(RAAS_E_UNSUPPORTED, "page = 1: the representative-key bound of one key is the key itself; use score_mode 0");
  if (c->page == 1 && c->quest_prefill_pages > 0)
    return fail(RAAS_E_UNSUPPORTED, "the Quest-on-prefill hybrid needs page = 16");
  if (c->head_dim != 64 && c->head_dim != 128)
    return fail(RAAS_E_UNSUPPORTED, "head_dim must be 64 or 128");
  d->g = c->n_q_heads / c->n_kv_heads;
  if (d->g > raas::MAX_GROUP) return fail(RAAS_E_UNSUPPORTED, "GQA group > 8");
  d->C = c->L / raas::PAGE;
  if (c->stamp_rule == 1 && d->Ce > 512)
    return fail(RAAS_E_UNSUPPORTED, "top-r stamping supports at most 512 pages (token slots) per unit");
  if (c->quest_prefill_pages < 0) return fail(RAAS_E_INVALID, "quest_prefill_pages must be >= 0");
  if (c->table_scope != 0 && c->table_scope != 1) return fail(RAAS_E_INVALID, "table_scope must be 0 or 1");
  if (c->disable_early_start != 0 && c->disable_early_start != 1)
    return fail(RAAS_E_INVALID, "disable_early_start must be 0 or 1");
  if (c->quest_prefill_pages > 0 && d->C > 512)
    return fail(RAAS_E_UNSUPPORTED, "the Quest-on-prefill hybrid supports L <= 8192 (512 pages)");
  d->units = c->batch * c->n_kv_heads;
  if (d->units >= (1 << 20)) return fail(RAAS_E_UNSUPPORTED, "more than 2^20 units per handle");
  if ((long long)d->units * d->C * raas::PAGE >= (1LL << 31))
    return fail(RAAS_E_UNSUPPORTED, "units * L too large for 32-bit TMA row coordinates");
  // auto: 32-page splits (the whole budget when L <= 512); depends on L only, never on batch
  int sp = c->split_pages > 0 ? c->split_pages : std::min(32, d->C);
  if (sp > 32) return fail(RAAS_E_UNSUPPORTED, "split_pages must be <= 32");
  const int min_sp = (d->C + raas::MAX_SPLITS - 1) / raas::MAX_SPLITS;
  if (sp < min_sp) sp = min_sp;
  if (sp > d->C) sp = d->C;
  if (sp > 32) return fail(RAAS_E_UNSUPPORTED, "L too large (more than 32*%d pages)", raas::MAX_SPLITS);
  d->split_pages = sp;
  d->nsplit = (d->C + sp - 1) / sp;
  return RAAS_OK;
}

Layout layout(const raas_config* c, const Derived& d) {
  Layout L{};
  const size_t U = d.units, C = d.C, D = c->head_dim, g = d.g;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = up(o + bytes); return r; };
  L.kvstore = take(U * C * d.pstr * 2);
  const size_t Ce = d.Ce;  // metadata entries (pages, or token slots when page = 1)
  L.ts = take(U * Ce * 4);
  L.start = take(U * Ce * 4);
  L.cnt = take(U * Ce * 4);
  L.npin = take(U * 4);
  L.nfull = take(U * 4);
  const bool hyb = c->quest_prefill_pages > 0;  // Quest-on-prefill hybrid workspace (NEXT-4)
  L.repkey = hyb ? take(U * C * 2 * D * 2) : 0;
  L.vmap = hyb ? take(U * C * 4) : 0;
  L.plen = take((size_t)c->batch * 4);
  L.plan = take(U * 16);
  L.counter = take(U * 4);
  L.req_x = c->table_scope ? take((size_t)c->batch * Ce * 4) : 0;   // zeroed by raas_create
  L.req_ctr = c->table_scope ? take((size_t)c->batch * 4) : 0;
  // per-row scores only for the non-deferred token path; pages keep one score per page
  L.pmax = take(d.tokd ? 16 : U * Ce * g * 4);
  L.q_prev = d.tokd ? take(U * g * D * 2) : 0;
  L.lse_prev = d.tokd ? take(U * 8 * 4) : 0;
  L.part_key = d.tokd ? take(U * d.nsplit * 16) : 0;
  L.part_acc = take(U * d.nsplit * g * D * 4);
  L.part_ml = take(U * d.nsplit * g * 8);
  L.status = take(16);
  L.sched = take(16);
  L.stats = take(64);
  L.sq = take(U * g * D * 2);
  L.sk = take(U * D * 2);
  L.sv = take(U * D * 2);
  L.so = take(U * g * D * 2);
  L.total = o;
  return L;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Host view: K and V stores [units][C][16][D] in logical order.  Device store: per page the 16
// K rows then the 16 V rows, each row keeping its 16-byte chunk c at chunk c ^ (row & 7) (see
// raas_kernels.cuh).  pack: logical -> device (k or v may be null: that half is left as is);
// unpack: device -> logical.
// (pstr: bf16 elements per device page, 2 * 16 * D plus the tokd trailer)
void pack_store(const uint16_t* k, const uint16_t* v, uint16_t* dev, size_t pages, int D, size_t pstr) {
  const int nch = D / 8;
  for (size_t pg = 0; pg < pages; ++pg)
    for (int half = 0; half < 2; ++half) {
      const uint16_t* src = half ? v : k;
      if (!src) continue;
      for (int r = 0; r < raas::PAGE; ++r) {
        const uint16_t* srow = src + (pg * raas::PAGE + r) * D;
        uint16_t* drow = dev + pg * pstr + (half * raas::PAGE + r) * D;
        for (int c = 0; c < nch; ++c) std::memcpy(drow + (c ^ (r & 7)) * 8, srow + c * 8, 16);
      }
    }
}
void unpack_store(const uint16_t* dev, uint16_t* k, uint16_t* v, size_t pages, int D, size_t pstr) {
  const int nch = D / 8;
  for (size_t pg = 0; pg < pages; ++pg)
    for (int half = 0; half < 2; ++half) {
      uint16_t* dst = half ? v : k;
      if (!dst) continue;
      for (int r = 0; r < raas::PAGE; ++r) {
        const uint16_t* srow = dev + pg * pstr + (half * raas::PAGE + r) * D;
        uint16_t* drow = dst + (pg * raas::PAGE + r) * D;
        for (int c = 0; c < nch; ++c) std::memcpy(drow + c * 8, srow + (c ^ (r & 7)) * 8, 16);
      }
    }
}

}  // namespace

#ifdef RAAS_DBG_TIMING
static int g_dbg_launch = 0;  // timeline slot of the next decode launch (debug builds)
#endif

struct raas_handle {
  raas_config cfg;
  Derived d;
  Layout lay;
  int device;
  int num_sms;
  int grid;
  int cl;  // cluster schedule (DecodeParams::cl): grid = units * nsplit, clusters of nsplit
  int half;  // half-size CTAs, two per SM (one-split units of the default method)
  int smem;
  uint8_t* arena;
  int prefilled;
  std::vector<int32_t> plen_host;  // prompt lengths, kept alive for the async upload
};

namespace {

// Last decode handle launched on each stream (early start, DecodeParams::early).  A decode
// kernel may read its handle's state before griddepcontrol.wait only if the kernel right before
// it in the stream is not this handle's previous step: every kernel of the PDL chain triggers
// its dependents after its own griddepcontrol.wait, so the kernel two back has completed.
// Kernels launched without PDL serialise fully, which is also safe.
std::mutex g_last_mu;
std::unordered_map<cudaStream_t, const raas_handle*> g_last_decode;

// true when the last decode launched on `st` is not h's (or there is none); no update
bool other_last(const raas_handle* h, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_last_mu);
  auto it = g_last_decode.find(st);
  return !(it != g_last_decode.end() && it->second == h);
}

bool note_launch(const raas_handle* h, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_last_mu);
  auto it = g_last_decode.find(st);
  const bool same = it != g_last_decode.end() && it->second == h;
  g_last_decode[st] = h;
  return !same;
}

template <int D>
int launch_decode(raas_handle* h, const void* q, const void* k_new, const void* v_new,
                  void* out, cudaStream_t st, bool after_copies = false) {
  DecodeParams p{};
  uint8_t* a = h->arena;
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.k_new = static_cast<const __nv_bfloat16*>(k_new);
  p.v_new = static_cast<const __nv_bfloat16*>(v_new);
  p.out = static_cast<__nv_bfloat16*>(out);
  p.kvstore = reinterpret_cast<__nv_bfloat16*>(a + h->lay.kvstore);
  p.ts = reinterpret_cast<int32_t*>(a + h->lay.ts);
  p.start = reinterpret_cast<int32_t*>(a + h->lay.start);
  p.cnt = reinterpret_cast<int32_t*>(a + h->lay.cnt);
  p.npin = reinterpret_cast<const int32_t*>(a + h->lay.npin);
  p.plan = reinterpret_cast<int4*>(a + h->lay.plan);
  p.counter = reinterpret_cast<int32_t*>(a + h->lay.counter);
  p.pmax = reinterpret_cast<float*>(a + h->lay.pmax);
  p.part_acc = reinterpret_cast<float*>(a + h->lay.part_acc);
  p.part_ml = reinterpret_cast<float2*>(a + h->lay.part_ml);
  p.status = reinterpret_cast<uint32_t*>(a + h->lay.status);
  p.sched = reinterpret_cast<int32_t*>(a + h->lay.sched);
  p.stats = reinterpret_cast<unsigned long long*>(a + h->lay.stats);
  p.units = h->d.units;
  p.C = h->d.C;
  p.Ce = h->d.Ce;
  p.ep = h->d.ep;
  p.tokd = h->d.tokd;
  p.pstr = h->d.pstr;
  p.q_prev = h->d.tokd ? reinterpret_cast<__nv_bfloat16*>(a + h->lay.q_prev) : nullptr;
  p.lse_prev = h->d.tokd ? reinterpret_cast<float*>(a + h->lay.lse_prev) : nullptr;
  p.part_key = h->d.tokd ? reinterpret_cast<int4*>(a + h->lay.part_key) : nullptr;
  p.nsplit = h->d.nsplit;
  p.split_pages = h->d.split_pages;
  p.g = h->d.g;
  p.score_mode = h->cfg.score_mode;
  p.stamp_rule = h->cfg.stamp_rule;
  p.top_r = h->cfg.top_r;
  p.quest_k = h->cfg.quest_prefill_pages;
  p.nfull = reinterpret_cast<const int32_t*>(a + h->lay.nfull);
  p.vmap = h->cfg.quest_prefill_pages > 0 ? reinterpret_cast<const int32_t*>(a + h->lay.vmap) : nullptr;
  p.table_scope = h->cfg.table_scope;
#ifdef RAAS_DBG_TIMING
  p.dbg_slot = g_dbg_launch++ & 7;
#endif
  {
    const bool other = note_launch(h, st);  // always record the launch
    // after_copies: staged cudaMemcpyAsync copies precede this launch (full serialisation).
    // The zero-copy ingest kernel triggers us at its start, so it does not count: the kernel
    // two back has completed, the one right before (this handle's or not) may still run.
    // the Quest-on-prefill hybrid's selection kernel (this handle's) runs right before the decode
    // kernel and writes the attended-page list: the producer issues only the pages that do not
    // depend on it before the wait; not when the caller opted out (raas.h "Early start")
    p.early = (other || after_copies) && !h->cfg.disable_early_start;
  }
  p.cl = h->cl;
  p.n_kv = h->cfg.n_kv_heads;
  p.req_x = h->cfg.table_scope ? reinterpret_cast<uint32_t*>(a + h->lay.req_x) : nullptr;
  p.req_ctr = h->cfg.table_scope ? reinterpret_cast<int32_t*>(a + h->lay.req_ctr) : nullptr;
  const float scale = h->cfg.softmax_scale > 0.f ? h->cfg.softmax_scale
                                                 : 1.0f / sqrtf((float)h->cfg.head_dim);
  p.scale_log2 = scale * 1.4426950408889634f;
  p.log2_alpha = h->cfg.alpha > 0.f ? log2f(h->cfg.alpha) : -INFINITY;

  if (p.quest_k > 0) {  // hybrid: this step's prompt-page selection from q (D24)
    const int units = h->d.units, C = h->d.C;
    cudaLaunchConfig_t qc{};
    qc.gridDim = dim3(units);
    qc.blockDim = dim3(raas::QSEL_THREADS);
    qc.dynamicSmemBytes = p.g * D * 4 + 9 * C + 16;
    qc.stream = st;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    qa[0].val.programmaticStreamSerializationAllowed = 1;
    qc.attrs = qa;
    qc.numAttrs = 1;
    RAAS_CUDA(cudaLaunchKernelEx(&qc, raas::raas_qselect_kernel<D>, p.q,
                                 reinterpret_cast<const __nv_bfloat16*>(a + h->lay.repkey), p.nfull,
                                 reinterpret_cast<int32_t*>(a + h->lay.vmap), units, C, p.g, p.quest_k));
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(h->grid);
  lc.blockDim = dim3(h->half ? LayHalf<D>::THREADS : Lay<D>::THREADS);
  lc.dynamicSmemBytes = h->smem;
  lc.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = h->cl ? h->d.nsplit : 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = h->cl ? 2 : 1;
  if (h->d.tokd)     RAAS_CUDA(cudaLaunchKernelEx(&lc, decode_kernel<D, true, false>(), p));
  else if (h->d.gen) RAAS_CUDA(cudaLaunchKernelEx(&lc, decode_kernel<D, false, true>(), p));
  else if (h->d.fm == raas::F_QUEST) RAAS_CUDA(cudaLaunchKernelEx(&lc, decode_kernel_f<D, raas::F_QUEST>(), p));
  else if (h->d.fm == raas::F_TOPR)  RAAS_CUDA(cudaLaunchKernelEx(&lc, decode_kernel_f<D, raas::F_TOPR>(), p));
  else if (h->d.fm == raas::F_TSC)   RAAS_CUDA(cudaLaunchKernelEx(&lc, decode_kernel_f<D, raas::F_TSC>(), p));
  else if (h->d.fm == raas::F_HYB)   RAAS_CUDA(cudaLaunchKernelEx(&lc, decode_kernel_f<D, raas::F_HYB>(), p));
  else if (h->cl)    RAAS_CUDA(cudaLaunchKernelEx(&lc, decode_kernel_cl<D>(), p));
  else if (h->half)  RAAS_CUDA(cudaLaunchKernelEx(&lc, decode_kernel_half<D>(), p));
  else               RAAS_CUDA(cudaLaunchKernelEx(&lc, decode_kernel<D, false, false>(), p));
  return RAAS_OK;
}

// Grid size for the unit-affine schedule (raas_decode.cuh TileSched): minimise the estimated
// critical path = the largest tile count of a CTA, plus, when some units are shared across CTAs,
// the cross-CTA combine that ends the kernel (~8 us, expressed in tiles of SP pages streamed at
// ~48 GB/s per SM: 8 KiB per page).  The result never changes numerics (the split arithmetic is
// schedule-free), only the speed.
int choose_grid(int units, int nsplit, int sp, int cap) {
  const long long tiles = (long long)units * nsplit;
  if (tiles <= 0) return 1;
  const double tile_us = sp * 8192.0 / 48e3;  // us per tile
  const double tail_tiles = 8.0 / tile_us;
  int best = 1;
  double best_cost = 1e30;
  const int hi = (int)std::min<long long>(cap, tiles);
  for (int G = 1; G <= hi; ++G) {
    const int fu = units / G, R = units - fu * G;
    const long long shared = (long long)R * nsplit;
    // units of one split are complete wherever they run (no cross-CTA combine)
    const double cost = (double)fu * nsplit + (double)((shared + G - 1) / G) +
                        (R > 0 && nsplit > 1 ? tail_tiles : 0.0);
    if (cost < best_cost - 1e-9 || (cost < best_cost + 1e-9 && G > best)) {
      best_cost = cost;
      best = G;
    }
  }
  return best;
}

template <int D, bool TOKD, bool GEN, int FM = 0>
int setup_kernel_t(raas_handle* h, bool want_cl) {
  auto k = want_cl ? decode_kernel_cl<D>() : FM ? decode_kernel_f<D, FM>() : decode_kernel<D, TOKD, GEN>();
  constexpr bool QTR = GEN || (FM & raas::F_QUEST);  // stages with room for the min / max rows
  h->smem = Lay<D, TOKD, QTR>::SMEM;
  RAAS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem));
  int per_sm = 0;
  RAAS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, Lay<D, TOKD, QTR>::THREADS, h->smem));
  if (per_sm < 1) return fail(RAAS_E_CUDA, "decode kernel does not fit on an SM");
  h->grid = choose_grid(h->d.units, h->d.nsplit, h->d.split_pages, h->num_sms * per_sm);
  if (const char* e = std::getenv("RAAS_GRID")) {  // tuning experiments only (scripts/)
    const int G = std::atoi(e);
    if (G > 0) h->grid = std::min(G, h->num_sms * per_sm);
  }
  // Cluster schedule when the (unit, split) tiles fit the SMs one per CTA and every unit is
  // split (small batches, e.g. config 2 at B = 1): each unit's nsplit CTAs form a cluster and
  // hand their split partials to the leader through distributed shared memory instead of L2
  // (publish + acq_rel counter + loads).  Numerics are the same as the default schedule's.
  h->cl = 0;
  const long long tiles = (long long)h->d.units * h->d.nsplit;
  if (want_cl && !GEN && !TOKD) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)tiles);
    lc.blockDim = dim3(Lay<D, TOKD, GEN>::THREADS);
    lc.dynamicSmemBytes = h->smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = h->d.nsplit;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, k, &lc) == cudaSuccess && nclusters > 0) {
      h->cl = 1;
      h->grid = (int)tiles;
    } else {
      cudaGetLastError();  // clusters of this size do not fit: keep the default schedule
    }
  }
  return RAAS_OK;
}
template <int D>
int setup_kernel(raas_handle* h) {
  if (h->d.tokd) return setup_kernel_t<D, true, false>(h, false);
  // cluster schedule (its own instantiation of the default method) when the (unit, split) tiles
  // fit the SMs one per CTA and every unit is split; RAAS_CLUSTER=0 disables it (A/B
  // experiments and the schedule-equivalence tests; numerics never depend on it)
  const long long tiles = (long long)h->d.units * h->d.nsplit;
  // the leader's receive area holds nsplit partials and the unit's page maxima [C][g] fp32,
  // and its combine's preloaded metadata covers C <= 32 * CLM pages
  const long long recv_need = (long long)h->d.nsplit * Lay<D>::RECV_SLOT + 4LL * h->d.C * h->d.g;
  bool want_cl = RAAS_CL && Lay<D>::CL_OK && !h->d.gen && !h->d.fm && h->d.nsplit >= 2 && h->d.nsplit <= 8 &&
                 tiles <= h->num_sms && recv_need <= (long long)NC * Lay<D>::DEPOSIT &&
                 h->d.C <= 32 * raas::CLM;
  if (const char* e = std::getenv("RAAS_CLUSTER")) want_cl = want_cl && std::atoi(e) != 0;
  if (h->d.gen) return setup_kernel_t<D, false, true>(h, false);
  if (h->d.fm == raas::F_QUEST) return setup_kernel_t<D, false, false, raas::F_QUEST>(h, false);
  if (h->d.fm == raas::F_TOPR) return setup_kernel_t<D, false, false, raas::F_TOPR>(h, false);
  if (h->d.fm == raas::F_TSC) return setup_kernel_t<D, false, false, raas::F_TSC>(h, false);
  if (h->d.fm == raas::F_HYB) return setup_kernel_t<D, false, false, raas::F_HYB>(h, false);
  if (want_cl) {
    int rc = setup_kernel_t<D, false, false>(h, true);
    if (rc || h->cl) return rc;  // else clusters of this size do not fit: default schedule
  }
  // units of one tile of <= 16 pages: L = 256 17.8 -> 17.0 us; 32-page tiles (L = 512) lose
  // (26.4 -> 27.2 us: 8 pages per consumer on half the consumers)
  bool want_half = h->d.nsplit == 1 && h->d.split_pages <= 16 && !h->d.fm;
  if (const char* e = std::getenv("RAAS_HALF")) want_half = want_half && std::atoi(e) != 0;  // A/B, tests
  if (want_half) {
    auto k = decode_kernel_half<D>();
    h->smem = LayHalf<D>::SMEM;
    RAAS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem));
    int per_sm = 0;
    RAAS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, LayHalf<D>::THREADS, h->smem));
    if (per_sm >= 2) {
      h->half = 1;
      h->grid = choose_grid(h->d.units, h->d.nsplit, h->d.split_pages, h->num_sms * per_sm);
      return RAAS_OK;
    }
  }
  return setup_kernel_t<D, false, false>(h, false);
}

int build_repkeys(raas_handle* h, cudaStream_t st) {
  if (h->cfg.quest_prefill_pages <= 0) return RAAS_OK;
  uint8_t* a = h->arena;
  const size_t total = (size_t)h->d.units * h->d.C * (h->cfg.head_dim / 8);
  const int blocks = (int)std::min<size_t>((total + 255) / 256, (size_t)h->num_sms * 16);
  auto* kvs = reinterpret_cast<const __nv_bfloat16*>(a + h->lay.kvstore);
  auto* rk = reinterpret_cast<__nv_bfloat16*>(a + h->lay.repkey);
  auto* nf = reinterpret_cast<const int32_t*>(a + h->lay.nfull);
  if (h->cfg.head_dim == 128)
    raas::raas_repkey_kernel<128><<<blocks, 256, 0, st>>>(kvs, rk, nf, h->d.units, h->d.C, h->d.pstr);
  else
    raas::raas_repkey_kernel<64><<<blocks, 256, 0, st>>>(kvs, rk, nf, h->d.units, h->d.C, h->d.pstr);
  RAAS_CUDA(cudaGetLastError());
  return RAAS_OK;
}

// Quest score mode: rebuild every page's min / max trailer from the store (after prefill /
// set_state; the decode kernel maintains them on write afterwards)
int build_qtrailers(raas_handle* h, cudaStream_t st) {
  if (!h->d.qtr) return RAAS_OK;
  uint8_t* a = h->arena;
  const size_t total = (size_t)h->d.units * h->d.C * (h->cfg.head_dim / 8);
  const int blocks = (int)std::min<size_t>((total + 255) / 256, (size_t)h->num_sms * 16);
  auto* kvs = reinterpret_cast<__nv_bfloat16*>(a + h->lay.kvstore);
  auto* cnt = reinterpret_cast<const int32_t*>(a + h->lay.cnt);
  if (h->cfg.head_dim == 128)
    raas::raas_qtrailer_kernel<128><<<blocks, 256, 0, st>>>(kvs, cnt, h->d.units, h->d.C, h->d.pstr);
  else
    raas::raas_qtrailer_kernel<64><<<blocks, 256, 0, st>>>(kvs, cnt, h->d.units, h->d.C, h->d.pstr);
  RAAS_CUDA(cudaGetLastError());
  return RAAS_OK;
}

int refresh(raas_handle* h, cudaStream_t st) {
  uint8_t* a = h->arena;
  const int wpb = 4;
  raas::raas_refresh<<<(h->d.units + wpb - 1) / wpb, 32 * wpb, 0, st>>>(
      reinterpret_cast<int32_t*>(a + h->lay.ts), reinterpret_cast<int32_t*>(a + h->lay.start),
      reinterpret_cast<int32_t*>(a + h->lay.cnt), reinterpret_cast<int32_t*>(a + h->lay.npin),
      reinterpret_cast<int4*>(a + h->lay.plan), reinterpret_cast<int32_t*>(a + h->lay.counter),
      reinterpret_cast<uint32_t*>(a + h->lay.status), h->d.units, h->d.Ce, h->d.ep, h->d.tokd);
  RAAS_CUDA(cudaGetLastError());
  return RAAS_OK;
}

// tokd: mirror the ts / start arrays into the pages' trailers (the decode kernel reads them
// with the page)
int tok_sync(raas_handle* h, cudaStream_t st) {
  if (!h->d.tokd) return RAAS_OK;
  uint8_t* a = h->arena;
  const size_t tiles = (size_t)h->d.units * h->d.C;
  const int blocks = (int)std::min<size_t>((tiles * 32 + 255) / 256, (size_t)h->num_sms * 8);
  raas::raas_tok_trailer_sync<<<blocks, 256, 0, st>>>(
      reinterpret_cast<__nv_bfloat16*>(a + h->lay.kvstore), reinterpret_cast<const int32_t*>(a + h->lay.ts),
      reinterpret_cast<const int32_t*>(a + h->lay.start), tiles, h->d.pstr);
  RAAS_CUDA(cudaGetLastError());
  return RAAS_OK;
}

// tokd: apply the stamp decisions still pending from the last step (before a state readout)
int tok_flush(raas_handle* h, cudaStream_t st) {
  if (!h->d.tokd || !h->prefilled) return RAAS_OK;
  uint8_t* a = h->arena;
  const float scale = h->cfg.softmax_scale > 0.f ? h->cfg.softmax_scale
                                                 : 1.0f / sqrtf((float)h->cfg.head_dim);
  const float l2a = h->cfg.alpha > 0.f ? log2f(h->cfg.alpha) : -INFINITY;
  auto* kvs = reinterpret_cast<__nv_bfloat16*>(a + h->lay.kvstore);
  auto* qp = reinterpret_cast<const __nv_bfloat16*>(a + h->lay.q_prev);
  auto* lp = reinterpret_cast<const float*>(a + h->lay.lse_prev);
  auto* ts = reinterpret_cast<int32_t*>(a + h->lay.ts);
  auto* np = reinterpret_cast<const int32_t*>(a + h->lay.npin);
  auto* pl = reinterpret_cast<int4*>(a + h->lay.plan);
  auto* stats = reinterpret_cast<unsigned long long*>(a + h->lay.stats);
  if (h->cfg.head_dim == 128)
    raas::raas_tok_flush<128><<<h->d.units, 256, 0, st>>>(kvs, qp, lp, ts, np, pl, stats, h->d.Ce,
                                                          h->d.g, scale * 1.4426950408889634f, l2a, h->d.pstr);
  else
    raas::raas_tok_flush<64><<<h->d.units, 256, 0, st>>>(kvs, qp, lp, ts, np, pl, stats, h->d.Ce,
                                                         h->d.g, scale * 1.4426950408889634f, l2a, h->d.pstr);
  RAAS_CUDA(cudaGetLastError());
  return RAAS_OK;
}

}  // namespace

extern "C" {

const char* raas_last_error(void) { return g_err; }

size_t raas_arena_bytes(const raas_config* cfg) {
  Derived d;
  if (derive(cfg, &d) != RAAS_OK) return 0;
  return layout(cfg, d).total;
}

int raas_create(const raas_config* cfg, void* arena, size_t arena_bytes, int device,
                raas_handle** out) {
  if (!out) return fail(RAAS_E_INVALID, "null output handle");
  *out = nullptr;
  Derived d;
  int rc = derive(cfg, &d);
  if (rc) return rc;
  Layout lay = layout(cfg, d);
  if (!arena || (reinterpret_cast<uintptr_t>(arena) & (ALIGN - 1)) != 0)
    return fail(RAAS_E_ARENA, "arena must be a 1024-byte aligned device pointer");
  if (arena_bytes < lay.total)
    return fail(RAAS_E_ARENA, "arena too small: %zu < %zu", arena_bytes, lay.total);
  DeviceGuard guard(device);
  raas_handle* h = new raas_handle();
  h->cfg = *cfg;
  h->d = d;
  h->lay = lay;
  h->device = device;
  h->arena = static_cast<uint8_t*>(arena);
  int sms = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    delete h;
    return fail(RAAS_E_CUDA, "cudaDeviceGetAttribute: %s", cudaGetErrorString(e));
  }
  h->num_sms = sms;
  rc = cfg->head_dim == 128 ? setup_kernel<128>(h) : setup_kernel<64>(h);
  if (!rc) {
    e = cudaMemset(arena, 0, lay.total);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = fail(RAAS_E_CUDA, "arena memset: %s", cudaGetErrorString(e));
  }
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return RAAS_OK;
}

int raas_destroy(raas_handle* h) {
  {
    std::lock_guard<std::mutex> lk(g_last_mu);
    for (auto it = g_last_decode.begin(); it != g_last_decode.end();)
      it = it->second == h ? g_last_decode.erase(it) : std::next(it);
  }
  delete h;
  return RAAS_OK;
}

int raas_prefill_varlen(raas_handle* h, const void* k, const void* v, const int32_t* P_host,
                        int32_t P_max, void* stream) {
  if (!h) return fail(RAAS_E_INVALID, "null handle");
  if (h->prefilled) return fail(RAAS_E_STATE, "handle already prefilled");
  if (!P_host || P_max < 0) return fail(RAAS_E_INVALID, "bad prompt lengths");
  const int B = h->cfg.batch;
  for (int b = 0; b < B; ++b) {
    if (P_host[b] < 0 || P_host[b] > P_max)
      return fail(RAAS_E_INVALID, "P[%d]=%d outside [0, P_max=%d]", b, P_host[b], P_max);
    const int Pp = (P_host[b] + h->d.ep - 1) / h->d.ep;
    if (Pp >= h->d.Ce)
      return fail(RAAS_E_BUDGET, "request %d: ceil(P/page)=%d leaves no decode entry (L/page=%d)", b, Pp,
                  h->d.Ce);
  }
  if (P_max > 0 && (!k || !v || !aligned16(k) || !aligned16(v)))
    return fail(RAAS_E_INVALID, "k/v must be non-null 16-byte aligned device pointers");
  DeviceGuard guard(h->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* a = h->arena;
  auto* kvs = reinterpret_cast<__nv_bfloat16*>(a + h->lay.kvstore);
  auto* plen = reinterpret_cast<int32_t*>(a + h->lay.plen);
  h->plen_host.assign(P_host, P_host + B);
  RAAS_CUDA(cudaMemcpyAsync(plen, h->plen_host.data(), (size_t)B * 4, cudaMemcpyHostToDevice, st));
  if (P_max > 0) {
    const size_t total = (size_t)h->d.units * P_max * (h->cfg.head_dim / 8);
    const int blocks = (int)std::min<size_t>((total + 255) / 256, (size_t)h->num_sms * 16);
    if (h->cfg.head_dim == 128)
      raas::raas_prefill_copy<128><<<blocks, 256, 0, st>>>(
          static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v), kvs, plen,
          h->d.units, h->cfg.n_kv_heads, P_max, h->d.C, h->d.pstr);
    else
      raas::raas_prefill_copy<64><<<blocks, 256, 0, st>>>(
          static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v), kvs, plen,
          h->d.units, h->cfg.n_kv_heads, P_max, h->d.C, h->d.pstr);
    RAAS_CUDA(cudaGetLastError());
  }
  const size_t n = (size_t)h->d.units * h->d.Ce;
  raas::raas_meta_init<<<(int)std::min<size_t>((n + 255) / 256, 4096), 256, 0, st>>>(
      reinterpret_cast<int32_t*>(a + h->lay.ts), reinterpret_cast<int32_t*>(a + h->lay.start),
      reinterpret_cast<int32_t*>(a + h->lay.cnt), reinterpret_cast<int32_t*>(a + h->lay.npin),
      reinterpret_cast<int32_t*>(a + h->lay.nfull), reinterpret_cast<int4*>(a + h->lay.plan), plen,
      h->d.units, h->cfg.n_kv_heads, h->d.Ce, h->d.ep);
  RAAS_CUDA(cudaGetLastError());
  int rc = build_repkeys(h, st);
  if (!rc) rc = build_qtrailers(h, st);
  if (!rc) rc = refresh(h, st);
  if (!rc) rc = tok_sync(h, st);
  if (rc) return rc;
  h->prefilled = 1;
  return RAAS_OK;
}

int raas_prefill(raas_handle* h, const void* k, const void* v, int32_t P, void* stream) {
  if (!h) return fail(RAAS_E_INVALID, "null handle");
  if (P < 0) return fail(RAAS_E_INVALID, "P < 0");
  std::vector<int32_t> plens((size_t)h->cfg.batch, P);
  return raas_prefill_varlen(h, k, v, plens.data(), P, stream);
}

int raas_decode_step(raas_handle* h, const void* q, const void* k_new, const void* v_new,
                     void* out, void* stream) {
  if (!h) return fail(RAAS_E_INVALID, "null handle");
  if (!h->prefilled) return fail(RAAS_E_STATE, "decode before prefill");
  if (!q || !k_new || !v_new || !out || !aligned16(q) || !aligned16(k_new) ||
      !aligned16(v_new) || !aligned16(out))
    return fail(RAAS_E_INVALID, "q/k_new/v_new/out must be non-null 16-byte aligned device pointers");
  DeviceGuard guard(h->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return h->cfg.head_dim == 128 ? launch_decode<128>(h, q, k_new, v_new, out, st)
                                : launch_decode<64>(h, q, k_new, v_new, out, st);
}

namespace {
// Device alias of a pinned, mapped host buffer (UVA: cudaHostAlloc / torch pin_memory), or
// nullptr for pageable memory or a misaligned pointer.
void* mapped_alias(const void* hp, uintptr_t align) {
  if (reinterpret_cast<uintptr_t>(hp) % align != 0) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, hp) != cudaSuccess) {
    cudaGetLastError();  // pageable memory on older drivers: clear the sticky-free error
    return nullptr;
  }
  if (at.type != cudaMemoryTypeHost || at.devicePointer == nullptr) return nullptr;
  return at.devicePointer;
}
}  // namespace

int raas_decode_step_host(raas_handle* h, const void* q_host, const void* k_new_host,
                          const void* v_new_host, void* out_host, void* stream) {
  if (!h) return fail(RAAS_E_INVALID, "null handle");
  if (!h->prefilled) return fail(RAAS_E_STATE, "decode before prefill");
  if (!q_host || !k_new_host || !v_new_host || !out_host)
    return fail(RAAS_E_INVALID, "null host buffer");
  DeviceGuard guard(h->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* a = h->arena;
  const size_t D = h->cfg.head_dim, U = h->d.units, g = h->d.g;
  const void* qm = mapped_alias(q_host, 16);
  const void* km = mapped_alias(k_new_host, 16);
  const void* vm = mapped_alias(v_new_host, 16);
  void* om = mapped_alias(out_host, 8);
#ifdef RAAS_DBG_E2E  // e2e breakdown experiment: 1 = out to device (no host write), 2 = no ingest
  static const int dbg_e2e = std::getenv("RAAS_DBG_E2E") ? std::atoi(std::getenv("RAAS_DBG_E2E")) : 0;
  if (dbg_e2e == 1) om = a + h->lay.so;
  if (dbg_e2e == 2) qm = km = vm = nullptr;
#endif
  if (qm && km && vm) {
    // pinned inputs: one zero-copy ingest kernel (PCIe reads overlap the previous kernel)
    const int nq = (int)(U * g * D * 2 / 16), nkv = (int)(U * D * 2 / 16);
    const int per_block = raas::INGEST_THREADS * raas::INGEST_PER;
    const int blocks = std::max(1, std::min(h->num_sms, (nq + 2 * nkv + per_block - 1) / per_block));
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(blocks);
    lc.blockDim = dim3(raas::INGEST_THREADS);
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    RAAS_CUDA(cudaLaunchKernelEx(&lc, raas::raas_ingest_kernel, static_cast<const uint4*>(qm),
                                 static_cast<const uint4*>(km), static_cast<const uint4*>(vm),
                                 reinterpret_cast<uint4*>(a + h->lay.sq), reinterpret_cast<uint4*>(a + h->lay.sk),
                                 reinterpret_cast<uint4*>(a + h->lay.sv), nq, nkv,
                                 other_last(h, st) ? 1 : 0));
  } else
#ifdef RAAS_DBG_E2E
  if (dbg_e2e != 2)
#endif
  {  // pageable inputs: staged copies
    RAAS_CUDA(cudaMemcpyAsync(a + h->lay.sq, q_host, U * g * D * 2, cudaMemcpyHostToDevice, st));
    RAAS_CUDA(cudaMemcpyAsync(a + h->lay.sk, k_new_host, U * D * 2, cudaMemcpyHostToDevice, st));
    RAAS_CUDA(cudaMemcpyAsync(a + h->lay.sv, v_new_host, U * D * 2, cudaMemcpyHostToDevice, st));
  }
  // pinned out: the combine stores the bf16 rows straight into host memory
  void* out = om ? om : a + h->lay.so;
  const bool copies = !(qm && km && vm);
  int rc = h->cfg.head_dim == 128
               ? launch_decode<128>(h, a + h->lay.sq, a + h->lay.sk, a + h->lay.sv, out, st, copies)
               : launch_decode<64>(h, a + h->lay.sq, a + h->lay.sk, a + h->lay.sv, out, st, copies);
  if (rc) return rc;
  if (!om) RAAS_CUDA(cudaMemcpyAsync(out_host, a + h->lay.so, U * g * D * 2, cudaMemcpyDeviceToHost, st));
  return RAAS_OK;
}

int raas_get_state(raas_handle* h, int32_t* t, int32_t* ts, int32_t* start_pos, int32_t* count,
                   uint8_t* pinned, void* stream) {
  if (!h) return fail(RAAS_E_INVALID, "null handle");
  DeviceGuard guard(h->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t U = h->d.units, C = h->d.Ce;  // metadata entries (pages, or token slots)
  if (int rc = tok_flush(h, st)) return rc;
  std::vector<int32_t> npin(U), nfull(U), vts(U * C);
  std::vector<int4> plan(U);
  uint8_t* a = h->arena;
  RAAS_CUDA(cudaMemcpyAsync(npin.data(), a + h->lay.npin, U * 4, cudaMemcpyDeviceToHost, st));
  RAAS_CUDA(cudaMemcpyAsync(nfull.data(), a + h->lay.nfull, U * 4, cudaMemcpyDeviceToHost, st));
  RAAS_CUDA(cudaMemcpyAsync(plan.data(), a + h->lay.plan, U * 16, cudaMemcpyDeviceToHost, st));
  RAAS_CUDA(cudaMemcpyAsync(vts.data(), a + h->lay.ts, U * C * 4, cudaMemcpyDeviceToHost, st));
  if (start_pos)
    RAAS_CUDA(cudaMemcpyAsync(start_pos, a + h->lay.start, U * C * 4, cudaMemcpyDeviceToHost, st));
  if (count)
    RAAS_CUDA(cudaMemcpyAsync(count, a + h->lay.cnt, U * C * 4, cudaMemcpyDeviceToHost, st));
  RAAS_CUDA(cudaStreamSynchronize(st));
  for (size_t u = 0; u < U; ++u) {
    if (t) t[u] = plan[u].w - 1;
    for (size_t p = 0; p < C; ++p) {
      const bool pin = (int)p < npin[u];
      if (ts) ts[u * C + p] = pin ? 0 : vts[u * C + p];
      // 1 = prompt page full at prefill, 2 = the prompt's partial last page (D13 / D24)
      if (pinned) pinned[u * C + p] = pin ? ((int)p < nfull[u] ? 1 : 2) : 0;
    }
  }
  return RAAS_OK;
}

int raas_set_state(raas_handle* h, const int32_t* t, const int32_t* ts, const int32_t* start_pos,
                   const int32_t* count, const uint8_t* pinned, const void* k_store_host,
                   const void* v_store_host, void* stream) {
  if (!h) return fail(RAAS_E_INVALID, "null handle");
  if (!t || !ts || !start_pos || !count || !pinned) return fail(RAAS_E_INVALID, "null state array");
  DeviceGuard guard(h->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t U = h->d.units, C = h->d.Ce;  // metadata entries (pages, or token slots)
  std::vector<int32_t> npin(U), nfull(U);
  std::vector<int4> plan(U);
  for (size_t u = 0; u < U; ++u) {
    int np = 0;
    while (np < (int)C && pinned[u * C + np]) ++np;
    for (size_t p = np; p < C; ++p)
      if (pinned[u * C + p]) return fail(RAAS_E_INVALID, "pinned pages must be a prefix (unit %zu)", u);
    // flag 2 marks the prompt's partial last page: only the last pinned page may carry it
    for (int p = 0; p + 1 < np; ++p)
      if (pinned[u * C + p] != 1)
        return fail(RAAS_E_INVALID, "pinned flag 2 (partial prompt page) on a page that is not the last pinned one (unit %zu)", u);
    if (np > 0 && pinned[u * C + np - 1] > 2) return fail(RAAS_E_INVALID, "pinned flag > 2 (unit %zu)", u);
    nfull[u] = (np > 0 && pinned[u * C + np - 1] == 2) ? np - 1 : np;
    bool hole = false;
    for (size_t p = 0; p < C; ++p) {
      if (count[u * C + p] < 0 || count[u * C + p] > h->d.ep)
        return fail(RAAS_E_INVALID, "count out of range");
      if (count[u * C + p] == 0) hole = true;
      else if (hole) return fail(RAAS_E_INVALID, "used pages must be a prefix (unit %zu)", u);
    }
    npin[u] = np;
    plan[u] = make_int4(0, 0, 0, t[u] + 1);
  }
  if (h->cfg.table_scope) {  // one table per request: the kv-heads' replicas must agree
    const size_t Hkv = h->cfg.n_kv_heads;
    for (size_t u = 0; u < U; ++u) {
      const size_t r = u - u % Hkv;
      if (u == r) continue;
      if (t[u] != t[r] || std::memcmp(ts + u * C, ts + r * C, C * 4) ||
          std::memcmp(start_pos + u * C, start_pos + r * C, C * 4) ||
          std::memcmp(count + u * C, count + r * C, C * 4) || std::memcmp(pinned + u * C, pinned + r * C, C))
        return fail(RAAS_E_INVALID, "table_scope 1: kv-head %zu of request %zu differs from kv-head 0",
                    u % Hkv, u / Hkv);
    }
  }
  uint8_t* a = h->arena;
  RAAS_CUDA(cudaMemcpyAsync(a + h->lay.ts, ts, U * C * 4, cudaMemcpyHostToDevice, st));
  RAAS_CUDA(cudaMemcpyAsync(a + h->lay.start, start_pos, U * C * 4, cudaMemcpyHostToDevice, st));
  RAAS_CUDA(cudaMemcpyAsync(a + h->lay.cnt, count, U * C * 4, cudaMemcpyHostToDevice, st));
  RAAS_CUDA(cudaMemcpyAsync(a + h->lay.npin, npin.data(), U * 4, cudaMemcpyHostToDevice, st));
  // the hybrid's selectable prompt pages: the pinned pages flagged 1 (D24)
  RAAS_CUDA(cudaMemcpyAsync(a + h->lay.nfull, nfull.data(), U * 4, cudaMemcpyHostToDevice, st));
  RAAS_CUDA(cudaMemcpyAsync(a + h->lay.plan, plan.data(), U * 16, cudaMemcpyHostToDevice, st));
  const size_t pages = U * h->d.C, D = h->cfg.head_dim;  // 16-row tiles
  std::vector<uint16_t> dev;
  if (k_store_host || v_store_host) {
    dev.resize(pages * h->d.pstr);
    if (!k_store_host || !v_store_host) {  // keep the half that is not replaced
      RAAS_CUDA(cudaMemcpyAsync(dev.data(), a + h->lay.kvstore, dev.size() * 2, cudaMemcpyDeviceToHost, st));
      RAAS_CUDA(cudaStreamSynchronize(st));
    }
    pack_store(static_cast<const uint16_t*>(k_store_host), static_cast<const uint16_t*>(v_store_host),
               dev.data(), pages, (int)D, h->d.pstr);
    RAAS_CUDA(cudaMemcpyAsync(a + h->lay.kvstore, dev.data(), dev.size() * 2, cudaMemcpyHostToDevice, st));
  }
  int rc = build_repkeys(h, st);
  if (!rc) rc = build_qtrailers(h, st);
  if (!rc) rc = refresh(h, st);
  if (!rc) rc = tok_sync(h, st);
  if (rc) return rc;
  RAAS_CUDA(cudaStreamSynchronize(st));
  h->prefilled = 1;
  return RAAS_OK;
}

int raas_get_kv(raas_handle* h, void* k_store_host, void* v_store_host, void* stream) {
  if (!h) return fail(RAAS_E_INVALID, "null handle");
  DeviceGuard guard(h->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t pages = (size_t)h->d.units * h->d.C;
  std::vector<uint16_t> dev(pages * h->d.pstr);
  RAAS_CUDA(cudaMemcpyAsync(dev.data(), h->arena + h->lay.kvstore, dev.size() * 2, cudaMemcpyDeviceToHost, st));
  RAAS_CUDA(cudaStreamSynchronize(st));
  unpack_store(dev.data(), static_cast<uint16_t*>(k_store_host), static_cast<uint16_t*>(v_store_host),
               pages, h->cfg.head_dim, h->d.pstr);
  return RAAS_OK;
}

int raas_get_status(raas_handle* h, void* stream) {
  if (!h) return -fail(RAAS_E_INVALID, "null handle");
  DeviceGuard guard(h->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t s = 0;
  if (cudaMemcpyAsync(&s, h->arena + h->lay.status, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return -fail(RAAS_E_CUDA, "status readback failed");
  return (int)s;
}

int raas_get_counters(raas_handle* h, uint64_t counters[4], void* stream) {
  if (!h || !counters) return fail(RAAS_E_INVALID, "null argument");
  DeviceGuard guard(h->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = tok_flush(h, st)) return rc;
  RAAS_CUDA(cudaMemcpyAsync(counters, h->arena + h->lay.stats, 32, cudaMemcpyDeviceToHost, st));
  RAAS_CUDA(cudaStreamSynchronize(st));
  return RAAS_OK;
}

#ifdef RAAS_DBG_TOKD_GLOBAL
RAAS_API int raas_debug_tokd(int32_t* out16) {
  return cudaMemcpyFromSymbol(out16, raas::g_tokd_dbg, 64) == cudaSuccess ? 0 : 1;
}
#endif
int raas_launch_info(const raas_handle* h, int32_t info[6]) {
  if (!h || !info) return fail(RAAS_E_INVALID, "null argument");
  info[0] = h->grid;
  info[1] = h->half ? (h->cfg.head_dim == 128 ? LayHalf<128>::THREADS : LayHalf<64>::THREADS)
                    : (h->cfg.head_dim == 128 ? Lay<128>::THREADS : Lay<64>::THREADS);
  info[2] = h->smem;
  info[3] = h->d.split_pages;
  info[4] = h->d.nsplit;
  info[5] = h->cl ? h->d.nsplit : 1;
  return RAAS_OK;
}

#ifdef RAAS_DBG_TIMING
// tuning experiment only (not part of the ABI in include/raas.h): read + clear the cycle counters
RAAS_API int raas_debug_units(uint64_t* out, int n) {
  RAAS_CUDA(cudaMemcpyFromSymbol(out, raas::g_raas_dbg_unit, sizeof(uint64_t) * (n < 4096 * 4 ? n : 4096 * 4)));
  if (n >= 4096 * 8)
    RAAS_CUDA(cudaMemcpyFromSymbol(out + 4096 * 4, raas::g_raas_dbg_comb, sizeof(uint64_t) * 4096 * 4));
  if (n >= 4096 * 16)
    RAAS_CUDA(cudaMemcpyFromSymbol(out + 4096 * 8, raas::g_raas_dbg_cyc, sizeof(uint64_t) * 4096 * 8));
  return RAAS_OK;
}
RAAS_API int raas_debug_timeline(uint64_t* out, int n) {  // [8][256][4], then cleared
  RAAS_CUDA(cudaMemcpyFromSymbol(out, raas::g_raas_tl, sizeof(uint64_t) * n));
  std::vector<uint64_t> z(8 * 256 * 4, 0);
  RAAS_CUDA(cudaMemcpyToSymbol(raas::g_raas_tl, z.data(), z.size() * 8));
  g_dbg_launch = 0;
  return RAAS_OK;
}
RAAS_API int raas_debug_timing(uint64_t* out, int n) {
  RAAS_CUDA(cudaMemcpyFromSymbol(out, raas::g_raas_dbg, sizeof(uint64_t) * n));
  std::vector<uint64_t> z(1024 * 16, 0);
  RAAS_CUDA(cudaMemcpyToSymbol(raas::g_raas_dbg, z.data(), z.size() * 8));
  return RAAS_OK;
}
#endif

}  // extern "C"
