/*
 * raas_ref.h — CPU ORACLE for the RaaS decode hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product (libraas, include/raas.h) never links,
 * includes or calls it, and it shares no code with the CUDA path.
 *
 * What it computes: page-based RaaS (§3.3 :143-151, App. B :358-398) one
 * decode step at a time, in fp64, following SURVEY.md §8(c1) step by step, with the
 * readings D1-D25 listed in DESIGN.md §3.  Every tensor is a HOST buffer; bf16 values
 * are passed as their raw uint16 bit patterns and widened exactly to double.
 *
 * Layouts (row-major):
 *   q, out      [batch][n_q_heads][head_dim]
 *   k, v        [batch][n_kv_heads][P][head_dim]       (prefill)
 *   k_new,v_new [batch][n_kv_heads][head_dim]
 *   state arrays [batch*n_kv_heads][C]  with C = L / page ("unit" = (request, kv-head))
 *
 * Return codes: 0 OK, 1 invalid argument, 3 state error (decode before prefill,
 * prefill twice), 4 budget (ceil(P/page) >= C, reading D14).
 */
#ifndef RAAS_REF_H
#define RAAS_REF_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t L;             /* token budget per unit, includes prefill (PAPER.md :173) */
  double  alpha;         /* stamp iff normalised score > alpha (:29, :169 default 1e-4) */
  int32_t page;          /* tokens per page (:147, 16); 1 = token-level RaaS of §3.2 */
  int32_t n_q_heads;
  int32_t n_kv_heads;
  int32_t head_dim;
  int32_t batch;
  double  softmax_scale; /* 0 => 1/sqrt(head_dim) */
  int32_t score_mode;    /* page score used for stamping:
                            0 = exact page max of the normalised scores (reading D4);
                            1 = Quest representative-key bound (§3.3 :147-151, App. B
                                :362): U_p = sum_c max(q_c min_c, q_c max_c) over the per-channel
                                min / max of the page's keys, estimated score exp(scale U_p - LSE)
                                (reading D22; "parity unpinned": the paper gives no formula) */
  int32_t stamp_rule;    /* 0 = stamp iff score > alpha; 1 = top-r (§3.2 :135): stamp
                            the k = ceilf(top_r * n) best-scored of the n unpinned resident pages,
                            ranked by (score desc, start_pos asc) (reading D23) */
  double  top_r;
  int32_t quest_prefill_pages; /* 0 = off.  K > 0: the Quest-on-prefill + RaaS-on-decode hybrid
                            (PAPER.md :173/:183, :237; reading D24): each step a unit attends
                            only the K full prompt pages with the largest representative-key
                            bound max_h sum_c max(q_hc min_c, q_hc max_c) (ties: lower page), plus
                            every other resident page; the prompt's KV stays resident */
  int32_t table_scope;   /* granularity of the page table (reading D5 / D25):
                            0 = one table per (request, kv-head), stamp if any q-head of the
                                GQA group exceeds the threshold (default);
                            1 = one table per request (per layer), shared by all its kv-heads:
                                a page is stamped if ANY of the request's q-heads exceeds it,
                                every kv-head evicts the same page.  The per-unit
                                state arrays then hold identical replicas. */
} raas_ref_config;

typedef struct raas_ref raas_ref;

int  raas_ref_create(const raas_ref_config* cfg, raas_ref** out);
void raas_ref_destroy(raas_ref* h);
int  raas_ref_prefill(raas_ref* h, const uint16_t* k, const uint16_t* v, int32_t P);
/* variable prompt lengths: k, v [batch][n_kv_heads][P_max][head_dim]; request b keeps its first
 * P[b] tokens.  raas_ref_prefill == every P[b] = P_max = P. */
int  raas_ref_prefill_varlen(raas_ref* h, const uint16_t* k, const uint16_t* v, const int32_t* P,
                             int32_t P_max);
/* one decode step for every unit; out may be NULL */
int  raas_ref_decode_step(raas_ref* h, const uint16_t* q, const uint16_t* k_new,
                          const uint16_t* v_new, double* out);
/* bookkeeping-only step (pin P5): slot selection + write as in decode_step, but the
 * stamp decisions are GIVEN: stamps[unit*C + p] != 0 stamps page p (ignored for pinned
 * or empty pages).  No K/V data is written or attended. */
int  raas_ref_step_stamps(raas_ref* h, const uint8_t* stamps);

/* state readout; any pointer may be NULL.  t[unit] = tokens so far (PAPER.md :394).
 * pinned[unit*C+p]: 0 = unpinned; 1 = prompt page full at prefill; 2 = the prompt's partial
 * last page (P % page != 0), which decode tokens fill (D13) and the hybrid never selects (D24). */
int  raas_ref_get_state(const raas_ref* h, int32_t* t, int32_t* ts, int32_t* start_pos,
                        int32_t* count, uint8_t* pinned);
/* lockstep resync (SURVEY §8c parity protocol): overwrite metadata and, when non-NULL,
 * the KV store (bf16 bits, [units][C][page][head_dim]).  cur/used are re-derived; the
 * hybrid's full prompt pages are the pages flagged 1 (see raas_ref_get_state). */
int  raas_ref_set_state(raas_ref* h, const int32_t* t, const int32_t* ts,
                        const int32_t* start_pos, const int32_t* count,
                        const uint8_t* pinned, const uint16_t* k_store,
                        const uint16_t* v_store);
/* KV store readout (bf16 bits, [units][C][page][head_dim]; never-written rows are 0);
 * either pointer may be NULL.  With raas_ref_get_state it is the whole resync state. */
int  raas_ref_get_kv(const raas_ref* h, uint16_t* k_store, uint16_t* v_store);
/* trace of the LAST step:
 *   evicted[unit]  = start_pos of the page evicted before attention, or -1
 *   slot[unit]     = page index the new token was written to
 *   pstar[unit*C+p]= max_{h in group, j in p} p_{h,j} for unpinned resident pages,
 *                    -1 otherwise (used for the |p*-alpha| exactness band) */
int  raas_ref_get_trace(const raas_ref* h, int32_t* evicted, int32_t* slot, double* pstar);
/* hybrid mode trace of the last step: attended[unit*C+p] (1 if page p was attended) and
 * qscore[unit*C+p] (the selection score of full prompt pages, -inf otherwise); either may be
 * NULL */
int  raas_ref_get_selection(const raas_ref* h, uint8_t* attended, double* qscore);
/* resident token positions of one unit after the last step, ascending; returns count */
int  raas_ref_resident_positions(const raas_ref* h, int32_t unit, int32_t* pos, int32_t cap);
/* threads used by the OpenMP loop over units (1 = serial); returns the effective count */
int  raas_ref_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
