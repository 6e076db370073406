/*
 * raas.h — libraas: the C ABI of the B200-native page-based RaaS decode hot path.
 *
 * RaaS = "Reasoning-Aware Attention Sparsity" (arXiv 2502.11147, /root/reference/PAPER.md).
 * One decode step of attention over a fixed budget of L KV-cache slots per
 * (request, kv-head) "unit", fused with the paper's bookkeeping:
 *   - the prompt's pages are pinned and never evicted ......... PAPER.md :29, :98, App. B :396
 *   - a page whose normalised attention score exceeds alpha gets
 *     the latest timestamp; time = number of tokens so far ...... :29, :98, :364, :394
 *   - when the cache is full the unpinned page with the oldest
 *     timestamp is evicted and the new K/V is written in place . :29, :98, :396; Fig 5 :100
 *   - pages of 16 tokens; one score per page .................. §3.3 :143-151
 * The readings adopted where the paper is silent (D1-D20: strict '>', per-(layer, kv-head)
 * tables with the score max-pooled over the GQA group, evict-before-attend order, ties to the
 * oldest page, ...) are listed in DESIGN.md §3 and SURVEY.md §8(c2).
 *
 * Conventions for every entry point:
 *   - All tensor pointers are CUDA DEVICE pointers unless the name says host; bf16 tensors are
 *     row-major and 16-byte aligned.  Layouts:
 *       q, out        [batch][n_q_heads][head_dim]            bf16
 *       k_new, v_new  [batch][n_kv_heads][head_dim]           bf16
 *       k, v (prefill)[batch][n_kv_heads][P][head_dim]        bf16
 *     A unit is u = b * n_kv_heads + kv_head.  q-head h reads kv-head h / (n_q/n_kv) (D15).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Ownership: the caller owns the arena (raas_arena_bytes() bytes of device memory, e.g.
 *     one torch.empty(..., dtype=uint8, device=...)) and every tensor; it must keep them
 *     alive until raas_destroy() and until the stream work using them has completed.  The
 *     library owns only the opaque host-side handle.  Nothing is allocated after create:
 *     memory is O(L) per unit for the life of the handle (PAPER.md :191-193).
 *   - Errors: an int status is returned.  Argument errors are detected synchronously and
 *     nothing is launched; device faults surface at the next synchronising call.  The
 *     thread-local message of the last failure is raas_last_error().
 *   - A handle is one attention layer of `batch` requests.  Handles are independent; a handle
 *     is not thread-safe.
 */
#ifndef RAAS_H
#define RAAS_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define RAAS_API __attribute__((visibility("default")))
#else
#define RAAS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define RAAS_OK             0
#define RAAS_E_INVALID      1  /* null/misaligned pointer, bad shape, L % page != 0, Hq % Hkv != 0 */
#define RAAS_E_UNSUPPORTED  2  /* head_dim not in {64,128}, page != 16, group > 8, budget too big */
#define RAAS_E_STATE        3  /* decode before prefill, prefill twice */
#define RAAS_E_BUDGET       4  /* ceil(P/page) >= L/page: no decode page left (reading D14) */
#define RAAS_E_CUDA         5  /* a CUDA call failed; see raas_last_error() */
#define RAAS_E_ARENA        6  /* arena too small or misaligned (needs 1024-byte alignment) */

typedef struct raas_handle raas_handle; /* opaque; one per (layer, request batch) */

typedef struct {
  int32_t L;             /* token budget per unit incl. prefill (PAPER.md :173, Fig 6 x-axis); L % page == 0 */
  float   alpha;         /* stamp iff normalised score > alpha (strict, D3); default 1e-4 (:169, D1).
                            0 stamps every page; >= 1 stamps none (StreamingLLM-like, :70) */
  int32_t page;          /* tokens per page; must be 16 (:147) */
  int32_t n_q_heads;     /* n_q_heads % n_kv_heads == 0, group n_q/n_kv <= 8 */
  int32_t n_kv_heads;
  int32_t head_dim;      /* 64 or 128 */
  int32_t batch;         /* requests held by this handle */
  float   softmax_scale; /* 0 => 1/sqrt(head_dim) */
  int32_t split_pages;   /* pages per split-K tile; 0 => auto (min(32, L/16), raised so L/16/split <= 80).
                            Independent of batch, so results are bitwise identical under
                            request sharding. */
  int32_t score_mode;    /* page score the stamp compares with alpha:
                            0 = exact page max of the normalised scores (reading D4, default);
                            1 = Quest representative-key bound, the paper's estimator (§3.3
                                :147-151, App. B :362): per channel c, max(q_c min_c, q_c max_c)
                                over the page's keys, summed, scaled and normalised by the step's
                                LSE (reading D22).  A superset of mode 0's stamps. */
  int32_t stamp_rule;    /* 0 = stamp iff score > alpha (the default, :29, :169);
                            1 = top-r (PAPER.md :135, "assign the latest timestamp to r=50% tokens
                                with the highest attention scores in each decoding step"): per
                                unit and step, the k = ceilf(top_r * n) highest-scored of the n
                                unpinned resident pages, ties to the oldest page (reading D23).
                                Needs L <= 8192. */
  float   top_r;         /* r in [0, 1] for stamp_rule 1 (0.5 in the paper) */
  int32_t quest_prefill_pages; /* 0 = off.  K > 0: the Quest-on-prefill + RaaS-on-decode hybrid
                            the paper recommends for long prompts / small budgets (:173, :183,
                            :237; reading D24).  Each step a unit attends only the K full prompt
                            pages with the largest representative-key bound
                            max_h sum_c max(q_c min_c, q_c max_c) (ties: lower page), plus all
                            other resident pages; stamping / eviction are unchanged (prompt pages
                            stay pinned and resident).  Adds one small launch per step
                            (bound + selection) and 1/16 of the prompt's K bytes.  L <= 8192.
                            With raas_set_state, the selectable pages are the pinned pages
                            flagged 1 (a flag-2 partial last prompt page is always attended). */
  int32_t table_scope;   /* page-table granularity (reading D25):
                            0 = one table per (request, kv-head), stamped when any q-head of the
                                GQA group exceeds the threshold (reading D5, default);
                            1 = one table per request (per layer handle), shared by all its
                                kv-heads: a page is stamped when ANY q-head of the request
                                exceeds it and every kv-head evicts the same page.  The state
                                arrays keep one identical replica per kv-head; raas_set_state
                                rejects replicas that differ.  Sharding a request's kv-heads over
                                handles would need an exchange, so shard by request only. */
  int32_t disable_early_start; /* 0 (default) = early start allowed, 1 = never (see "Early start"
                            below); changes timing only, never results */
} raas_config;

/* Bytes of device memory the handle needs (KV store: per unit L/16 pages, each 16 K rows + 16 V
 * rows of head_dim bf16, int32 page metadata, L2-resident split-K workspace, staging for raas_decode_step_host).
 * O(L) per unit, fixed for the life of the handle.  Returns 0 for an invalid config. */
RAAS_API size_t raas_arena_bytes(const raas_config* cfg);

/* Validate cfg, carve the arena (device pointer, >= raas_arena_bytes, 1024-byte aligned) on
 * CUDA device `device`, zero it, build the TMA descriptors.  Synchronous. */
RAAS_API int raas_create(const raas_config* cfg, void* arena, size_t arena_bytes, int device,
                raas_handle** out);

/* Store the prompt's K/V (P tokens per unit, positions 1..P) into pages 0..ceil(P/16)-1,
 * which are pinned (App. B :396); time t = P (:394).  Asynchronous on `stream`.
 * Errors: RAAS_E_STATE if already prefilled, RAAS_E_BUDGET if ceil(P/16) >= L/16.
 * The prompt's attention output is not computed here (that is the model's prefill). */
RAAS_API int raas_prefill(raas_handle* h, const void* k, const void* v, int32_t P, void* stream);

/* Variable prompt lengths: request b's prompt is the first P_host[b] tokens of
 * k, v laid out [batch][n_kv_heads][P_max][head_dim] (the rest is padding, never read).  Each
 * request gets its own pinned pages and clock (t = P_host[b]).  P_host is a host array of
 * `batch` int32; it is copied into the handle, so it may be released on return.  Errors as
 * raas_prefill, RAAS_E_BUDGET if any request's prompt leaves it no decode page.
 * raas_prefill(h, k, v, P, s) is raas_prefill_varlen with every P_host[b] = P_max = P. */
RAAS_API int raas_prefill_varlen(raas_handle* h, const void* k, const void* v, const int32_t* P_host,
                                 int32_t P_max, void* stream);

/* Early start (programmatic dependent launch, PDL).  raas_decode_step launches with the
 * programmatic-stream-serialization attribute and calls griddepcontrol.launch_dependents right
 * after its own griddepcontrol.wait.  When the kernel right before it in the stream is NOT this
 * handle's previous decode step (the usual case: one handle per layer, layers interleaved on one
 * stream), the kernel reads its handle's state (write plan, page counts) and issues its first
 * K/V page copies BEFORE griddepcontrol.wait, overlapping the previous kernel's tail.  This is
 * safe because the handle's previous step then completed before the previous kernel could
 * trigger this one.  CONTRACT for callers that enable it (the default):
 *   - every PDL kernel placed on the same stream between two steps of one handle must trigger
 *     its dependents only after its own griddepcontrol.wait (standard practice; a kernel that
 *     triggers earlier could let a decode step read state its own previous step is still
 *     writing);
 *   - nothing but libraas may write a handle's arena between its steps (raas_set_state and
 *     raas_prefill are stream-ordered and reset the tracking).
 * The library tracks, per stream, the last handle it launched a decode step for; a handle
 * stepped twice in a row waits as usual.  Set cfg.disable_early_start = 1 to never read state
 * before griddepcontrol.wait (e.g. when foreign PDL kernels that trigger early share the
 * stream).  The Quest-on-prefill hybrid never starts early (its selection kernel, launched right
 * before the step, writes the attended-page list). */

/* One decode step for every unit of the handle:
 *   t += 1; pick the slot (current page, else a fresh page, else the victim chosen at the end
 *   of the previous step = argmin over unpinned pages of (ts, start_pos)); write k_new/v_new
 *   there; out = softmax(scale q K^T) V over every resident token incl. the new one; stamp
 *   ts = t on each unpinned page p with max_{h in group, j in p} (s_hj - LSE_h) > ln(alpha);
 *   pre-select the next victim.
 * One kernel launch, no host synchronisation, CUDA-graph capturable (t, the write cursor and
 * the victim live on the device).  Errors: RAAS_E_STATE before prefill. */
RAAS_API int raas_decode_step(raas_handle* h, const void* q, const void* k_new, const void* v_new,
                     void* out, void* stream);

/* Same step with HOST buffers (same layouts).  Pinned (page-locked, mapped: cudaHostAlloc,
 * torch pin_memory) inputs are read over PCIe by a small ingest kernel that runs ahead of the
 * step (the host reads overlap the previous kernel of the stream), and a pinned `out_host` is
 * written directly by the step's combine (zero-copy); pageable buffers go through async
 * staging copies in the arena.  Either way the result is bitwise that of raas_decode_step.
 * Host buffers must hold the step's data when the call is made (pinned inputs may be read
 * before earlier work in the stream completes) and stay valid until the stream completes. */
RAAS_API int raas_decode_step_host(raas_handle* h, const void* q_host, const void* k_new_host,
                          const void* v_new_host, void* out_host, void* stream);

/* Release the host handle.  Does not free the arena (the caller owns it). */
RAAS_API int raas_destroy(raas_handle* h);

/* ---- introspection / test support (synchronise `stream`) ---- */

/* Host copies of the page metadata: t[units] (tokens so far), ts/start_pos/count [units][L/16]
 * int32, pinned [units][L/16] uint8: 0 = unpinned, 1 = a prompt page that was full at prefill,
 * 2 = the prompt's partial last page (P % 16 != 0: decode tokens fill it and it stays pinned,
 * reading D13; the Quest-on-prefill hybrid never drops it, D24).  Pinned pages report ts = 0
 * (D17).  Any output may be NULL. */
RAAS_API int raas_get_state(raas_handle* h, int32_t* t, int32_t* ts, int32_t* start_pos, int32_t* count,
                   uint8_t* pinned, void* stream);

/* Lockstep resync (SURVEY.md §8c parity protocol): overwrite the metadata (host arrays in the
 * raas_get_state layout; pinned pages must be a prefix 0..Pp-1 of each unit, only the last of
 * them may carry flag 2, decode pages must be the pages that follow) and, if non-NULL, the KV
 * store from host bf16 arrays [units][L/16][16][head_dim].  The write cursor (the used page
 * with the largest start position) and the next victim are re-derived on the device, so
 * get_state -> set_state continues bitwise as the uninterrupted run.  Marks the handle
 * prefilled.  RAAS_E_INVALID on a malformed state (nothing is written). */
RAAS_API int raas_set_state(raas_handle* h, const int32_t* t, const int32_t* ts, const int32_t* start_pos,
                   const int32_t* count, const uint8_t* pinned, const void* k_store_host,
                   const void* v_store_host, void* stream);

/* Host copy of the KV store, bf16 [units][L/16][16][head_dim] each (either may be NULL). */
RAAS_API int raas_get_kv(raas_handle* h, void* k_store_host, void* v_store_host, void* stream);

/* Device-side status word (0 = OK; bit 0: a step found no evictable page).  Synchronises. */
RAAS_API int raas_get_status(raas_handle* h, void* stream);

/* Cumulative counters since create, summed over units: [0] page stamps, [1] stamp decisions
 * (unpinned resident pages examined), [2] evictions, [3] unit-steps.  Synchronises. */
RAAS_API int raas_get_counters(raas_handle* h, uint64_t counters[4], void* stream);

/* Launch shape of the decode kernel (for roofline accounting): grid CTAs, threads per CTA,
 * dynamic shared memory bytes, split pages, splits per unit, thread-block cluster size (1: the
 * default persistent schedule; nsplit: the cluster schedule for small batches, where each
 * unit's split CTAs exchange their partials through distributed shared memory). */
RAAS_API int raas_launch_info(const raas_handle* h, int32_t info[6]);

/* Thread-local message describing the last error (never NULL). */
RAAS_API const char* raas_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RAAS_H */
