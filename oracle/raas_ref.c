/*
 * raas_ref.c — CPU ORACLE for page-based RaaS decode.  TEST INFRASTRUCTURE ONLY
 * (see raas_ref.h).  Plain, slow, fp64, one unit at a time; no blocking, no fusion,
 * no streaming softmax.  Each block cites the passage it follows.
 *
 * Algorithm (readings D1-D25 in DESIGN.md §3):
 *   prefill(P):  pages 0..Pp-1 hold positions 1..P in order, 16 per page; they are
 *                pinned ("Pages corresponding to prefill tokens are exempt from
 *                eviction", App. B :396); t = P (time = number of tokens,
 *                :394).
 *   decode step: t += 1                                   (:394; Fig 5 row 5 -> ts 5, :100)
 *                slot = current page if not full, else a fresh page if the budget
 *                allows, else evict argmin_{unpinned} (ts, start_pos)
 *                                                         (:29, :98 "evict tokens with the
 *                                                          oldest timestamp"; :396; D9-D12)
 *                write k,v; a written unpinned page gets ts = t (D8)
 *                attend over all resident tokens          (standard attention, :46-48, :70)
 *                stamp every unpinned page holding a token with normalised score > alpha
 *                                                         (:29, :98, :364; D2-D5)
 */
#include "raas_ref.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { REF_OK = 0, REF_E_INVALID = 1, REF_E_STATE = 3, REF_E_BUDGET = 4 };

typedef struct {
  int32_t *start, *count, *ts;
  uint8_t *pinned;
  double *K, *V;          /* [C][page][d] */
  int32_t used, cur, t;
  int32_t evicted, slot;  /* trace of the last step */
  double *pstar;          /* [C] */
  int32_t nfull;          /* full prompt pages (selectable in the hybrid mode) */
  uint8_t *attended;      /* [C] hybrid trace */
  double *qscore;         /* [C] hybrid trace */
  double *best;           /* [C] decisive log-score of the last step (before the stamp) */
} ref_unit;

struct raas_ref {
  raas_ref_config cfg;
  int32_t C, units, g;
  double scale;
  int prefilled;
  ref_unit* u;
};

static int g_threads = 1;

int raas_ref_set_threads(int n) {
#ifdef _OPENMP
  if (n <= 0) n = omp_get_num_procs();
  g_threads = n;
#else
  (void)n;
  g_threads = 1;
#endif
  return g_threads;
}

/* bf16 bit pattern -> exact double (bf16 is the top half of an IEEE binary32). */
static double widen_bf16(uint16_t b) {
  uint32_t x = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &x, sizeof f);
  return (double)f;
}

int raas_ref_create(const raas_ref_config* cfg, raas_ref** out) {
  if (!cfg || !out) return REF_E_INVALID;
  if (cfg->L <= 0 || cfg->page <= 0 || cfg->L % cfg->page != 0) return REF_E_INVALID;
  if (cfg->n_q_heads <= 0 || cfg->n_kv_heads <= 0 || cfg->n_q_heads % cfg->n_kv_heads != 0)
    return REF_E_INVALID;
  if (cfg->head_dim <= 0 || cfg->batch <= 0) return REF_E_INVALID;
  if (!(cfg->alpha >= 0.0)) return REF_E_INVALID;
  if (cfg->score_mode != 0 && cfg->score_mode != 1) return REF_E_INVALID;
  if (cfg->stamp_rule != 0 && cfg->stamp_rule != 1) return REF_E_INVALID;
  if (cfg->stamp_rule == 1 && !(cfg->top_r >= 0.0 && cfg->top_r <= 1.0)) return REF_E_INVALID;
  if (cfg->quest_prefill_pages < 0) return REF_E_INVALID;
  if (cfg->table_scope != 0 && cfg->table_scope != 1) return REF_E_INVALID;
  raas_ref* h = (raas_ref*)calloc(1, sizeof *h);
  if (!h) return REF_E_INVALID;
  h->cfg = *cfg;
  h->C = cfg->L / cfg->page;
  h->units = cfg->batch * cfg->n_kv_heads;
  h->g = cfg->n_q_heads / cfg->n_kv_heads;
  h->scale = cfg->softmax_scale != 0.0 ? cfg->softmax_scale : 1.0 / sqrt((double)cfg->head_dim);
  h->u = (ref_unit*)calloc((size_t)h->units, sizeof(ref_unit));
  size_t kv = (size_t)h->C * cfg->page * cfg->head_dim;
  for (int32_t i = 0; i < h->units; ++i) {
    ref_unit* u = &h->u[i];
    u->start = (int32_t*)calloc((size_t)h->C, sizeof(int32_t));
    u->count = (int32_t*)calloc((size_t)h->C, sizeof(int32_t));
    u->ts = (int32_t*)calloc((size_t)h->C, sizeof(int32_t));
    u->pinned = (uint8_t*)calloc((size_t)h->C, 1);
    u->pstar = (double*)calloc((size_t)h->C, sizeof(double));
    u->attended = (uint8_t*)calloc((size_t)h->C, 1);
    u->qscore = (double*)calloc((size_t)h->C, sizeof(double));
    u->best = (double*)calloc((size_t)h->C, sizeof(double));
    u->K = (double*)calloc(kv, sizeof(double));
    u->V = (double*)calloc(kv, sizeof(double));
    u->cur = -1;
    u->evicted = -1;
    u->slot = -1;
  }
  *out = h;
  return REF_OK;
}

void raas_ref_destroy(raas_ref* h) {
  if (!h) return;
  for (int32_t i = 0; i < h->units; ++i) {
    ref_unit* u = &h->u[i];
    free(u->start); free(u->count); free(u->ts); free(u->pinned);
    free(u->pstar); free(u->K); free(u->V); free(u->attended); free(u->qscore);
    free(u->best);
  }
  free(h->u);
  free(h);
}

/* Prefill (§2.1 :46 "computing and caching the key and value vectors for each
 * token"; App. B :396 prefill pages exempt).  Positions 1..P_b, 16 per page (:147); request b
 * keeps the first P[b] of its P_max rows. */
int raas_ref_prefill_varlen(raas_ref* h, const uint16_t* k, const uint16_t* v, const int32_t* P,
                            int32_t P_max) {
  if (!h || !P || P_max < 0 || (P_max > 0 && (!k || !v))) return REF_E_INVALID;
  if (h->prefilled) return REF_E_STATE;
  const int32_t page = h->cfg.page, d = h->cfg.head_dim, C = h->C;
  for (int32_t b = 0; b < h->cfg.batch; ++b) {
    if (P[b] < 0 || P[b] > P_max) return REF_E_INVALID;
    if ((P[b] + page - 1) / page >= C) return REF_E_BUDGET;  /* D14: a decode page per unit */
  }
  for (int32_t ui = 0; ui < h->units; ++ui) {
    ref_unit* u = &h->u[ui];
    const int32_t Pu = P[ui / h->cfg.n_kv_heads];
    const int32_t Pp = (Pu + page - 1) / page;
    for (int32_t j = 0; j < Pu; ++j) {            /* token j has position j+1 */
      int32_t p = j / page, off = j % page;
      for (int32_t c = 0; c < d; ++c) {
        u->K[((size_t)p * page + off) * d + c] = widen_bf16(k[((size_t)ui * P_max + j) * d + c]);
        u->V[((size_t)p * page + off) * d + c] = widen_bf16(v[((size_t)ui * P_max + j) * d + c]);
      }
    }
    for (int32_t p = 0; p < Pp; ++p) {
      u->start[p] = p * page + 1;
      u->count[p] = (Pu - p * page) < page ? (Pu - p * page) : page;
      u->ts[p] = 0;                               /* D17: pinned pages' ts untracked */
      u->pinned[p] = 1;
    }
    u->used = Pp;
    u->cur = Pp - 1;                              /* -1 when P == 0 */
    u->t = Pu;
    u->nfull = Pu / page;
    u->evicted = -1;
    u->slot = -1;
  }
  h->prefilled = 1;
  return REF_OK;
}

int raas_ref_prefill(raas_ref* h, const uint16_t* k, const uint16_t* v, int32_t P) {
  if (!h || P < 0) return REF_E_INVALID;
  int32_t* Ps = (int32_t*)malloc(sizeof(int32_t) * (size_t)h->cfg.batch);
  for (int32_t b = 0; b < h->cfg.batch; ++b) Ps[b] = P;
  const int rc = raas_ref_prefill_varlen(h, k, v, Ps, P);
  free(Ps);
  return rc;
}

/* Slot selection and in-place write for one unit (D9-D13).
 * Returns the slot; records the eviction. */
static int32_t select_and_write(raas_ref* h, ref_unit* u, const uint16_t* kn, const uint16_t* vn) {
  const int32_t page = h->cfg.page, d = h->cfg.head_dim, C = h->C;
  u->t += 1;                                      /* time counts this token (:394) */
  u->evicted = -1;
  int32_t slot;
  if (u->cur >= 0 && u->count[u->cur] < page) {
    slot = u->cur;                                /* keep filling (also D13) */
  } else {
    if (u->used < C) {
      slot = u->used;                             /* budget not reached (:100 first steps) */
      u->used += 1;
    } else {
      /* "When the cache is full, we evict tokens with the oldest timestamp" (:29, :98);
       * prefill exempt (:396); ties -> smallest start_pos (D12). */
      slot = -1;
      for (int32_t p = 0; p < C; ++p) {
        if (u->pinned[p]) continue;
        if (slot < 0 || u->ts[p] < u->ts[slot] ||
            (u->ts[p] == u->ts[slot] && u->start[p] < u->start[slot]))
          slot = p;
      }
      u->evicted = u->start[slot];
    }
    u->count[slot] = 0;                           /* the evicted tokens vanish here (D9) */
    u->pinned[slot] = 0;
    u->start[slot] = u->t;
  }
  int32_t off = u->count[slot];
  if (kn && vn) {
    for (int32_t c = 0; c < d; ++c) {
      u->K[((size_t)slot * page + off) * d + c] = widen_bf16(kn[c]);
      u->V[((size_t)slot * page + off) * d + c] = widen_bf16(vn[c]);
    }
  }
  u->count[slot] += 1;
  if (!u->pinned[slot]) u->ts[slot] = u->t;       /* a written page carries its write time (D8) */
  u->cur = slot;
  u->slot = slot;
  return slot;
}

static void decode_unit(raas_ref* h, int32_t ui, const uint16_t* q, const uint16_t* k_new,
                        const uint16_t* v_new, double* out) {
  const int32_t page = h->cfg.page, d = h->cfg.head_dim, C = h->C, g = h->g;
  const int32_t Hq = h->cfg.n_q_heads, Hkv = h->cfg.n_kv_heads;
  const int32_t b = ui / Hkv, kvh = ui % Hkv;
  ref_unit* u = &h->u[ui];
  select_and_write(h, u, k_new + (size_t)ui * d, v_new + (size_t)ui * d);

  double* s = (double*)malloc((size_t)C * page * sizeof(double));
  double* best = u->best;
  double* qh = (double*)malloc((size_t)d * sizeof(double));
  for (int32_t p = 0; p < C; ++p) best[p] = -INFINITY;

  /* which pages this step attends: all resident pages, except that the hybrid mode keeps only
   * the K best full prompt pages by Quest's representative-key bound (D24) */
  const int32_t Kq = h->cfg.quest_prefill_pages;
  for (int32_t p = 0; p < C; ++p) {
    u->attended[p] = u->count[p] > 0;
    u->qscore[p] = -INFINITY;
  }
  if (Kq > 0 && u->nfull > Kq) {
    for (int32_t p = 0; p < u->nfull; ++p) {
      double sc = -INFINITY;
      for (int32_t hh = 0; hh < g; ++hh) {
        const int32_t qi = b * Hq + kvh * g + hh;
        double U = 0.0;
        for (int32_t c = 0; c < d; ++c) {
          double mn = INFINITY, mxk = -INFINITY;
          for (int32_t i = 0; i < u->count[p]; ++i) {
            const double kc = u->K[((size_t)p * page + i) * d + c];
            if (kc < mn) mn = kc;
            if (kc > mxk) mxk = kc;
          }
          const double qc = widen_bf16(q[(size_t)qi * d + c]);
          U += (qc * mn > qc * mxk) ? qc * mn : qc * mxk;
        }
        if (U > sc) sc = U;
      }
      u->qscore[p] = sc;
      u->attended[p] = 0;
    }
    for (int32_t r = 0; r < Kq; ++r) {            /* top-K by (score desc, page asc) */
      int32_t arg = -1;
      for (int32_t p = 0; p < u->nfull; ++p) {
        if (u->attended[p]) continue;
        if (arg < 0 || u->qscore[p] > u->qscore[arg]) arg = p;
      }
      u->attended[arg] = 1;
    }
  }

  for (int32_t hh = 0; hh < g; ++hh) {            /* q-head h uses kv-head floor(h/g) (D15) */
    const int32_t qi = b * Hq + kvh * g + hh;
    for (int32_t c = 0; c < d; ++c) qh[c] = widen_bf16(q[(size_t)qi * d + c]);
    /* scores s_j = scale * <q, k_j> over every resident token (D2, D20) */
    double mx = -INFINITY;
    for (int32_t p = 0; p < C; ++p)
      for (int32_t i = 0; i < (u->attended[p] ? u->count[p] : 0); ++i) {
        const double* kj = &u->K[((size_t)p * page + i) * d];
        double acc = 0.0;
        for (int32_t c = 0; c < d; ++c) acc += qh[c] * kj[c];
        s[p * page + i] = h->scale * acc;
        if (s[p * page + i] > mx) mx = s[p * page + i];
      }
    /* LSE = log sum_j exp(s_j)  (softmax normaliser, :70) */
    double sum = 0.0;
    for (int32_t p = 0; p < C; ++p)
      for (int32_t i = 0; i < (u->attended[p] ? u->count[p] : 0); ++i) sum += exp(s[p * page + i] - mx);
    const double lse = mx + log(sum);
    if (out) {
      double* o = out + (size_t)qi * d;
      for (int32_t c = 0; c < d; ++c) o[c] = 0.0;
      for (int32_t p = 0; p < C; ++p)
        for (int32_t i = 0; i < (u->attended[p] ? u->count[p] : 0); ++i) {
          const double w = exp(s[p * page + i] - lse);
          const double* vj = &u->V[((size_t)p * page + i) * d];
          for (int32_t c = 0; c < d; ++c) o[c] += w * vj[c];
        }
    }
    /* decisive log-score per page, max over the heads of the group (D5):
     *  mode 0: exact page max of the normalised scores (D4);
     *  mode 1: Quest's bound -- "a representative key (K) for each page ... the query (Q) ...
     *          attends to these representative keys to compute a single attention score per
     *          page" (:147-151, :362): per channel c, max(q_c * min_j k_jc, q_c * max_j k_jc)
     *          summed over c, scaled, normalised by the step's LSE (D22). */
    for (int32_t p = 0; p < C; ++p) {
      if (u->pinned[p] || u->count[p] == 0) continue;
      double lp = -INFINITY;
      if (h->cfg.score_mode == 0) {
        for (int32_t i = 0; i < u->count[p]; ++i)
          if (s[p * page + i] - lse > lp) lp = s[p * page + i] - lse;
      } else {
        double U = 0.0;
        for (int32_t c = 0; c < d; ++c) {
          double mn = INFINITY, mx = -INFINITY;
          for (int32_t i = 0; i < u->count[p]; ++i) {
            const double kc = u->K[((size_t)p * page + i) * d + c];
            if (kc < mn) mn = kc;
            if (kc > mx) mx = kc;
          }
          const double a = qh[c] * mn, b = qh[c] * mx;
          U += a > b ? a : b;
        }
        lp = h->scale * U - lse;
      }
      if (lp > best[p]) best[p] = lp;
    }
  }
  free(s); free(qh);
}

/* a6 for one unit, given the decisive log-score best[p] of every page: the unit's own
 * (table_scope 0) or the maximum over the request's kv-heads (table_scope 1, D25). */
static void stamp_unit(raas_ref* h, ref_unit* u, const double* best) {
  const int32_t C = h->C;
  /* stamp: "we assign it the latest timestamp" when the score is above alpha (:29, :98,
   * :364), strictly (D3), in the log domain s - LSE > ln(alpha) (D2). */
  const double ln_alpha = log(h->cfg.alpha);     /* alpha = 0 -> -inf: every page stamped */
  if (h->cfg.stamp_rule == 0) {
    for (int32_t p = 0; p < C; ++p) {
      u->pstar[p] = -1.0;
      if (u->pinned[p] || u->count[p] == 0) continue;
      u->pstar[p] = exp(best[p]);
      if (best[p] > ln_alpha) u->ts[p] = u->t;
    }
  } else {
    /* top-r (:135): "assign the latest timestamp to r=50% tokens with the highest attention
     * scores in each decoding step", at page level over the unpinned resident pages (D23):
     * k = ceilf(r * n) pages, ranked by score, ties to the smaller start_pos.  Selection by
     * repeated maximum (plain, O(n k)). */
    int32_t n = 0;
    for (int32_t p = 0; p < C; ++p) {
      u->pstar[p] = -1.0;
      if (u->pinned[p] || u->count[p] == 0) continue;
      u->pstar[p] = exp(best[p]);
      n++;
    }
    int32_t k = (int32_t)ceilf((float)h->cfg.top_r * (float)n);
    if (k > n) k = n;
    uint8_t* taken = (uint8_t*)calloc((size_t)C, 1);
    for (int32_t r = 0; r < k; ++r) {
      int32_t arg = -1;
      for (int32_t p = 0; p < C; ++p) {
        if (u->pinned[p] || u->count[p] == 0 || taken[p]) continue;
        if (arg < 0 || best[p] > best[arg] || (best[p] == best[arg] && u->start[p] < u->start[arg]))
          arg = p;
      }
      taken[arg] = 1;
      u->ts[arg] = u->t;
    }
    free(taken);
  }
}

int raas_ref_decode_step(raas_ref* h, const uint16_t* q, const uint16_t* k_new,
                         const uint16_t* v_new, double* out) {
  if (!h || !q || !k_new || !v_new) return REF_E_INVALID;
  if (!h->prefilled) return REF_E_STATE;
  int32_t ui;
#pragma omp parallel for schedule(static) num_threads(g_threads)
  for (ui = 0; ui < h->units; ++ui) decode_unit(h, ui, q, k_new, v_new, out);
  if (h->cfg.table_scope == 0) {
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (ui = 0; ui < h->units; ++ui) stamp_unit(h, &h->u[ui], h->u[ui].best);
  } else {
    /* one page table per request: "tokens" of the layer are stamped when any head's score
     * exceeds alpha (reading D25 of :29, :98 at request granularity) */
    const int32_t Hkv = h->cfg.n_kv_heads, C = h->C;
    double* rb = (double*)malloc((size_t)C * sizeof(double));
    for (int32_t b = 0; b < h->cfg.batch; ++b) {
      for (int32_t p = 0; p < C; ++p) {
        rb[p] = -INFINITY;
        for (int32_t kv = 0; kv < Hkv; ++kv)
          if (h->u[b * Hkv + kv].best[p] > rb[p]) rb[p] = h->u[b * Hkv + kv].best[p];
      }
      for (int32_t kv = 0; kv < Hkv; ++kv) stamp_unit(h, &h->u[b * Hkv + kv], rb);
    }
    free(rb);
  }
  return REF_OK;
}

int raas_ref_step_stamps(raas_ref* h, const uint8_t* stamps) {
  if (!h || !stamps) return REF_E_INVALID;
  if (!h->prefilled) return REF_E_STATE;
  for (int32_t ui = 0; ui < h->units; ++ui) {
    ref_unit* u = &h->u[ui];
    select_and_write(h, u, NULL, NULL);
    for (int32_t p = 0; p < h->C; ++p) {
      u->pstar[p] = -1.0;
      if (u->pinned[p] || u->count[p] == 0) continue;
      if (stamps[(size_t)ui * h->C + p]) u->ts[p] = u->t;
    }
  }
  return REF_OK;
}

int raas_ref_get_state(const raas_ref* h, int32_t* t, int32_t* ts, int32_t* start_pos,
                       int32_t* count, uint8_t* pinned) {
  if (!h) return REF_E_INVALID;
  const int32_t C = h->C;
  for (int32_t ui = 0; ui < h->units; ++ui) {
    const ref_unit* u = &h->u[ui];
    if (t) t[ui] = u->t;
    if (ts) memcpy(ts + (size_t)ui * C, u->ts, (size_t)C * sizeof(int32_t));
    if (start_pos) memcpy(start_pos + (size_t)ui * C, u->start, (size_t)C * sizeof(int32_t));
    if (count) memcpy(count + (size_t)ui * C, u->count, (size_t)C * sizeof(int32_t));
    /* pinned flags: 1 = a prompt page that was full at prefill (selectable by the hybrid, D24),
     * 2 = the prompt's partial last page (P % page != 0; decode tokens fill it, D13) */
    if (pinned)
      for (int32_t p = 0; p < C; ++p)
        pinned[(size_t)ui * C + p] = u->pinned[p] ? (p < u->nfull ? 1 : 2) : 0;
  }
  return REF_OK;
}

/* bf16 bits of a double that holds an exact bf16 value (every stored K/V element does) */
static uint16_t narrow_bf16(double x) {
  const float f = (float)x;
  uint32_t b;
  memcpy(&b, &f, sizeof b);
  return (uint16_t)(b >> 16);
}

int raas_ref_get_kv(const raas_ref* h, uint16_t* k_store, uint16_t* v_store) {
  if (!h) return REF_E_INVALID;
  const size_t kv = (size_t)h->C * h->cfg.page * h->cfg.head_dim;
  for (int32_t ui = 0; ui < h->units; ++ui)
    for (size_t i = 0; i < kv; ++i) {
      if (k_store) k_store[(size_t)ui * kv + i] = narrow_bf16(h->u[ui].K[i]);
      if (v_store) v_store[(size_t)ui * kv + i] = narrow_bf16(h->u[ui].V[i]);
    }
  return REF_OK;
}

int raas_ref_set_state(raas_ref* h, const int32_t* t, const int32_t* ts,
                       const int32_t* start_pos, const int32_t* count, const uint8_t* pinned,
                       const uint16_t* k_store, const uint16_t* v_store) {
  if (!h || !t || !ts || !start_pos || !count || !pinned) return REF_E_INVALID;
  const int32_t C = h->C, page = h->cfg.page, d = h->cfg.head_dim;
  const size_t kv = (size_t)C * page * d;
  for (int32_t ui = 0; ui < h->units; ++ui) {
    ref_unit* u = &h->u[ui];
    u->t = t[ui];
    memcpy(u->ts, ts + (size_t)ui * C, (size_t)C * sizeof(int32_t));
    memcpy(u->start, start_pos + (size_t)ui * C, (size_t)C * sizeof(int32_t));
    memcpy(u->count, count + (size_t)ui * C, (size_t)C * sizeof(int32_t));
    u->nfull = 0;
    for (int32_t p = 0; p < C; ++p) {
      u->pinned[p] = pinned[(size_t)ui * C + p] != 0;
      if (pinned[(size_t)ui * C + p] == 1) u->nfull += 1;  /* flag 1: full prompt page (D24) */
    }
    u->used = 0;
    u->cur = -1;
    for (int32_t p = 0; p < C; ++p) {
      if (u->count[p] > 0) {
        u->used += 1;
        if (u->cur < 0 || u->start[p] > u->start[u->cur]) u->cur = p;
      }
    }
    if (k_store)
      for (size_t i = 0; i < kv; ++i) u->K[i] = widen_bf16(k_store[(size_t)ui * kv + i]);
    if (v_store)
      for (size_t i = 0; i < kv; ++i) u->V[i] = widen_bf16(v_store[(size_t)ui * kv + i]);
    u->evicted = -1;
    u->slot = -1;
  }
  h->prefilled = 1;
  return REF_OK;
}

int raas_ref_get_trace(const raas_ref* h, int32_t* evicted, int32_t* slot, double* pstar) {
  if (!h) return REF_E_INVALID;
  for (int32_t ui = 0; ui < h->units; ++ui) {
    const ref_unit* u = &h->u[ui];
    if (evicted) evicted[ui] = u->evicted;
    if (slot) slot[ui] = u->slot;
    if (pstar) memcpy(pstar + (size_t)ui * h->C, u->pstar, (size_t)h->C * sizeof(double));
  }
  return REF_OK;
}

int raas_ref_get_selection(const raas_ref* h, uint8_t* attended, double* qscore) {
  if (!h) return REF_E_INVALID;
  for (int32_t ui = 0; ui < h->units; ++ui) {
    if (attended) memcpy(attended + (size_t)ui * h->C, h->u[ui].attended, (size_t)h->C);
    if (qscore) memcpy(qscore + (size_t)ui * h->C, h->u[ui].qscore, (size_t)h->C * sizeof(double));
  }
  return REF_OK;
}

int raas_ref_resident_positions(const raas_ref* h, int32_t unit, int32_t* pos, int32_t cap) {
  if (!h || unit < 0 || unit >= h->units) return -1;
  const ref_unit* u = &h->u[unit];
  int32_t n = 0;
  /* gather, then insertion-sort ascending (tiny sizes only) */
  for (int32_t p = 0; p < h->C; ++p)
    for (int32_t i = 0; i < u->count[p]; ++i) {
      if (n < cap && pos) pos[n] = u->start[p] + i;
      n++;
    }
  if (pos) {
    int32_t m = n < cap ? n : cap;
    for (int32_t a = 1; a < m; ++a) {
      int32_t x = pos[a], b = a - 1;
      while (b >= 0 && pos[b] > x) { pos[b + 1] = pos[b]; --b; }
      pos[b + 1] = x;
    }
  }
  return n;
}
