"""Seeded synthetic inputs for the RaaS decode path (shared by tests, oracle runs, bench).

This module holds NO arithmetic of the method (no attention, no timestamps, no
eviction): it only draws q / k / v streams and rounds them to bf16.  Both the CUDA path
and the CPU oracle consume exactly the bf16 bit patterns produced here.

Recipes:

* ``gaussian_stream`` — i.i.d. N(0, sigma^2) q/k/v.  Page-level stamping is ~100% on this
  data, so it exercises the attention numerics, not the eviction policy.
* ``waterfall_stream`` — the "waterfall" pattern of PAPER.md §3.1 (:27, :88-94, Fig 3
  :108): a sink page (the "lazy" StreamingLLM pattern, >70% of maps), the two most
  recent pages, milestone decode pages that emerge and fade (20-25% of maps; decay
  half-life 256 steps) and rare phoenix reactivations of prefill pages (1-2%, gaps >128
  steps).  Keys of one logical page share a signature vector, so page-level stamping
  is selective (30-60% of pages at the calibrated lambda), which is what makes eviction
  non-trivial.
"""
from __future__ import annotations

import math

import numpy as np

PAGE = 16


def bf16_bits(x) -> np.ndarray:
    """Round float32 -> bf16 (round-to-nearest-even) and return the uint16 bit patterns."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    nan = np.isnan(f)
    out = rounded.astype(np.uint16)
    if nan.any():
        out[nan] = 0x7FC0
    return out


def bf16_to_f32(bits) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(bits, dtype=np.uint16))
    return (b.astype(np.uint32) << 16).view(np.float32)


class Stream:
    """A full decode workload: prefill K/V plus T steps of (q, k_new, v_new), as bf16 bits.

    Shapes: k_pre, v_pre [B, Hkv, P, d]; q [T, B, Hq, d]; k, v [T, B, Hkv, d].
    """

    def __init__(self, k_pre, v_pre, q, k, v):
        self.k_pre, self.v_pre, self.q, self.k, self.v = k_pre, v_pre, q, k, v

    @property
    def T(self):
        return self.q.shape[0]

    @property
    def P(self):
        return self.k_pre.shape[2]


def gaussian_stream(seed, B, Hq, Hkv, d, P, T, sigma_q=1.0, sigma_k=1.0, sigma_v=1.0) -> Stream:
    rng = np.random.Generator(np.random.Philox(seed))
    k_pre = bf16_bits(rng.standard_normal((B, Hkv, P, d), np.float32) * sigma_k)
    v_pre = bf16_bits(rng.standard_normal((B, Hkv, P, d), np.float32) * sigma_v)
    q = bf16_bits(rng.standard_normal((T, B, Hq, d), np.float32) * sigma_q)
    k = bf16_bits(rng.standard_normal((T, B, Hkv, d), np.float32) * sigma_k)
    v = bf16_bits(rng.standard_normal((T, B, Hkv, d), np.float32) * sigma_v)
    return Stream(k_pre, v_pre, q, k, v)


def waterfall_stream(seed, B, Hq, Hkv, d, P, T, lam=6.0, eta=1.0, key_noise=0.5,
                     p_milestone=0.1, milestone_half_life=256.0, p_phoenix=1.0 / 512,
                     phoenix_len=32, recent_weight=0.8, phoenix_weight=0.8) -> Stream:
    """Waterfall-shaped stream (§3.1, Fig 3).  Positions are 1-based; the
    logical page of position j is (j-1)//16 (a property of the workload, not of the
    cache: the generator does not know what the cache retained)."""
    rng = np.random.Generator(np.random.Philox(seed))
    g = Hq // Hkv
    U = B * Hkv
    n_tok = P + T
    n_pages = (n_tok + PAGE - 1) // PAGE
    phi = rng.standard_normal((U, n_pages, d)).astype(np.float64)
    phi /= np.linalg.norm(phi, axis=-1, keepdims=True)
    page_of = np.arange(n_tok) // PAGE                       # position j+1 -> page
    keys = phi[:, page_of, :] + key_noise * rng.standard_normal((U, n_tok, d)) / np.sqrt(d)
    vals = rng.standard_normal((U, n_tok, d))
    pp = (P + PAGE - 1) // PAGE                              # pages touched by the prompt
    # milestones: a page that starts inside the decode becomes one with prob p_milestone
    first_pos = np.arange(n_pages) * PAGE + 1
    is_dec_page = first_pos > P
    ms = (rng.random((U, n_pages)) < p_milestone) & is_dec_page[None, :]
    ms_strength = rng.uniform(0.2, 1.0, (U, n_pages)) * ms
    phoenix_until = np.full(U, -1, np.int64)
    phoenix_page = np.zeros(U, np.int64)
    q = np.empty((T, B, Hq, d), np.float32)
    for i in range(T):
        t = P + i + 1                                        # position of the new token
        cur = (t - 1) // PAGE
        w = np.zeros((U, n_pages))
        w[:, 0] = 1.0                                        # sink ("lazy" maps)
        w[:, cur] = np.maximum(w[:, cur], recent_weight)
        if cur >= 1:
            w[:, cur - 1] = np.maximum(w[:, cur - 1], recent_weight)
        age = t - first_pos[None, : cur + 1]
        decay = np.where(age >= 0, 2.0 ** (-np.maximum(age, 0) / milestone_half_life), 0.0)
        w[:, : cur + 1] = np.maximum(w[:, : cur + 1], ms_strength[:, : cur + 1] * decay)
        if pp > 0:
            start = (rng.random(U) < p_phoenix) & (phoenix_until < t)
            phoenix_page[start] = rng.integers(0, pp, int(start.sum()))
            phoenix_until[start] = t + phoenix_len
            act = phoenix_until >= t
            w[act, phoenix_page[act]] = np.maximum(w[act, phoenix_page[act]], phoenix_weight)
        base = lam * np.sqrt(d) * np.einsum("up,upd->ud", w, phi)
        noise = eta * rng.standard_normal((U, g, d))
        q[i] = (base[:, None, :] + noise).reshape(B, Hkv * g, d)
    keys = keys.reshape(B, Hkv, n_tok, d).astype(np.float32)
    vals = vals.reshape(B, Hkv, n_tok, d).astype(np.float32)
    k_pre = bf16_bits(keys[:, :, :P])
    v_pre = bf16_bits(vals[:, :, :P])
    k = bf16_bits(np.moveaxis(keys[:, :, P:], 2, 0))
    v = bf16_bits(np.moveaxis(vals[:, :, P:], 2, 0))
    return Stream(k_pre, v_pre, bf16_bits(q), k, v)


def random_steady_state(seed, units, C, Pp, t_now, page=PAGE):
    """A full-cache state for bounded-sample timing (bench CPU baseline): pinned prefill
    pages 0..Pp-1, C-Pp full decode pages of 16 consecutive positions each, the newest
    one ending at t_now, timestamps in [end of page, t_now].  Draws numbers only; the
    method's rules are not applied here.  Requires t_now >= Pp*page + 4*page*(C-Pp)."""
    nd = C - Pp
    assert t_now >= Pp * page + 4 * page * nd, "t_now too small for the spread"
    rng = np.random.Generator(np.random.Philox(seed))
    ts = np.zeros((units, C), np.int32)
    start = np.zeros((units, C), np.int32)
    count = np.full((units, C), page, np.int32)
    pinned = np.zeros((units, C), np.uint8)
    pinned[:, :Pp] = 1
    start[:, :Pp] = np.arange(Pp) * page + 1
    for u in range(units):
        offs = np.concatenate([[0], np.sort(rng.choice(np.arange(1, 4 * nd), nd - 1, replace=False))])
        starts = t_now - page + 1 - page * offs
        ts_u = np.minimum(t_now, starts + page - 1 + rng.integers(0, 64, nd))
        ts_u[0] = t_now
        perm = rng.permutation(nd)
        start[u, Pp:] = starts[perm]
        ts[u, Pp:] = ts_u[perm]
    t = np.full(units, t_now, np.int32)
    return dict(t=t, ts=ts, start=start, count=count, pinned=pinned)


class WaterfallTorch:
    """The ``waterfall_stream`` recipe drawn on a torch device, step by step, for the bench.

    Same workload structure as ``waterfall_stream`` (sink page, the two most recent pages,
    milestone decode pages decaying with a 256-step half-life, phoenix prefill
    reactivations; keys share their logical page's signature), drawn with torch's Philox
    generator so that full-size workloads (512 units x 16k steps) need no host round trip.
    The bit patterns differ from ``waterfall_stream`` (different RNG); the oracle never
    consumes this stream.  Inputs only: no attention, timestamps or eviction here.
    """

    def __init__(self, seed, B, Hq, Hkv, d, P, T_max, device, lam=6.0, eta=1.0, key_noise=0.5,
                 p_milestone=0.1, milestone_half_life=256.0, p_phoenix=1.0 / 512,
                 phoenix_len=32, recent_weight=0.8, phoenix_weight=0.8):
        import torch

        self.torch = torch
        self.B, self.Hq, self.Hkv, self.d, self.P = B, Hq, Hkv, d, P
        self.g = Hq // Hkv
        self.U = B * Hkv
        self.dev = torch.device(device)
        self.gen = torch.Generator(device=self.dev)
        self.gen.manual_seed(seed)
        self.lam, self.eta, self.key_noise = lam, eta, key_noise
        self.half_life, self.p_phoenix, self.phoenix_len = milestone_half_life, p_phoenix, phoenix_len
        self.recent_weight, self.phoenix_weight = recent_weight, phoenix_weight
        self.n_pages = (P + T_max + PAGE - 1) // PAGE
        phi = torch.randn((self.U, self.n_pages, d), device=self.dev, generator=self.gen)
        self.phi = phi / phi.norm(dim=-1, keepdim=True)
        self.first_pos = torch.arange(self.n_pages, device=self.dev, dtype=torch.float32) * PAGE + 1
        is_dec = self.first_pos > P
        ms = (torch.rand((self.U, self.n_pages), device=self.dev, generator=self.gen) < p_milestone) & is_dec
        self.ms_strength = (0.2 + 0.8 * torch.rand((self.U, self.n_pages), device=self.dev,
                                                    generator=self.gen)) * ms
        self.pp = (P + PAGE - 1) // PAGE
        self.phoenix_until = torch.full((self.U,), -1, device=self.dev, dtype=torch.int64)
        self.phoenix_page = torch.zeros((self.U,), device=self.dev, dtype=torch.int64)
        self.i = 0                                      # decode steps drawn so far

    def prefill(self, chunk=4096):
        """Prompt K/V, bf16 [B, Hkv, P, d] (drawn in chunks of positions)."""
        torch = self.torch
        B, Hkv, P, d = self.B, self.Hkv, self.P, self.d
        k = torch.empty((B, Hkv, P, d), device=self.dev, dtype=torch.bfloat16)
        v = torch.empty_like(k)
        kf, vf = k.view(self.U, P, d), v.view(self.U, P, d)
        for a in range(0, P, chunk):
            b = min(P, a + chunk)
            pg = torch.arange(a, b, device=self.dev) // PAGE
            z = torch.randn((self.U, b - a, d), device=self.dev, generator=self.gen)
            kf[:, a:b] = (self.phi[:, pg] + self.key_noise * z / math.sqrt(d)).bfloat16()
            vf[:, a:b] = torch.randn((self.U, b - a, d), device=self.dev, generator=self.gen).bfloat16()
        return k, v

    def step(self, q_out, k_out, v_out):
        """Draw decode step i (new token at position t = P + i + 1) into bf16 tensors
        q_out [B, Hq, d], k_out / v_out [B, Hkv, d] (on the current stream)."""
        torch = self.torch
        t = self.P + self.i + 1
        cur = (t - 1) // PAGE
        assert cur < self.n_pages, "T_max exceeded"
        U, d = self.U, self.d
        age = t - self.first_pos[: cur + 1]
        decay = torch.where(age >= 0, torch.exp2(-age.clamp(min=0) / self.half_life), 0.0)
        w = self.ms_strength[:, : cur + 1] * decay
        w[:, 0] = torch.clamp(w[:, 0], min=1.0)                       # sink ("lazy" maps)
        w[:, cur] = torch.clamp(w[:, cur], min=self.recent_weight)    # the two most recent pages
        if cur >= 1:
            w[:, cur - 1] = torch.clamp(w[:, cur - 1], min=self.recent_weight)
        if self.pp > 0:                                               # phoenix reactivations
            start = (torch.rand((U,), device=self.dev, generator=self.gen) < self.p_phoenix) \
                & (self.phoenix_until < t)
            pick = torch.randint(0, self.pp, (U,), device=self.dev, generator=self.gen)
            self.phoenix_page = torch.where(start, pick, self.phoenix_page)
            self.phoenix_until = torch.where(start, torch.full_like(self.phoenix_until, t + self.phoenix_len),
                                             self.phoenix_until)
            act = (self.phoenix_until >= t).float() * self.phoenix_weight
            rows = torch.arange(U, device=self.dev)
            w[rows, self.phoenix_page] = torch.maximum(w[rows, self.phoenix_page], act)
        base = (self.lam * math.sqrt(d)) * torch.bmm(w[:, None, :], self.phi[:, : cur + 1]).squeeze(1)
        noise = self.eta * torch.randn((U, self.g, d), device=self.dev, generator=self.gen)
        q_out.view(U, self.g, d).copy_(base[:, None, :] + noise)
        z = torch.randn((U, d), device=self.dev, generator=self.gen)
        k_out.view(U, d).copy_(self.phi[:, cur] + self.key_noise * z / math.sqrt(d))
        v_out.view(U, d).copy_(torch.randn((U, d), device=self.dev, generator=self.gen))
        self.i += 1


def waterfall_resume(seed, B, Hq, Hkv, d, L, P, T, cur_count=5, lam=6.0, eta=1.0, key_noise=0.5,
                     p_milestone=0.1, milestone_half_life=256.0, p_phoenix=1.0 / 512,
                     phoenix_len=32, recent_weight=0.8, phoenix_weight=0.8, span=4):
    """A full-cache state in the middle of a long waterfall decode, plus the next T steps.

    For the full-size parity runs (configs 2-5), which cannot afford the oracle over the whole
    fill: every unit holds its prompt pages (pinned) and C - Pp decode pages of logical pages of
    the waterfall workload (``waterfall_stream``'s recipe: page signatures phi, keys
    phi + key_noise z / sqrt(d), queries lam sqrt(d) sum_p w_p(t) phi_p + eta zeta with the sink,
    the two most recent pages, decaying milestones and phoenix prompt pages).  The write page is
    the current logical page m_cur holding ``cur_count`` tokens (1..16; < 16: a partial current
    page), so t_now = 16 m_cur + cur_count.  The other resident decode pages are drawn among the
    ``span`` * (C - Pp) logical pages before m_cur, the milestone pages preferred (what a
    retention policy keeps), in random slots; their timestamps are drawn in [last position,
    t_now].  Draws numbers only: no attention, stamping or eviction rule is applied.

    Returns (state dict(t, ts, start, count, pinned) [units][C], k_store, v_store bf16 bits
    [units][C][16][d], Stream with k_pre/v_pre = None and T steps of q / k / v)."""
    assert P % PAGE == 0, "prompt pages are full here"
    assert 1 <= cur_count <= PAGE
    rng = np.random.Generator(np.random.Philox(seed))
    g, U = Hq // Hkv, B * Hkv
    C, Pp = L // PAGE, P // PAGE
    nd = C - Pp
    assert nd >= 2
    m_cur = Pp + span * nd                                   # logical page of token t_now
    t_now = PAGE * m_cur + cur_count
    n_pages = m_cur + (cur_count + T) // PAGE + 2
    phi = rng.standard_normal((U, n_pages, d), dtype=np.float32)
    phi /= np.linalg.norm(phi, axis=-1, keepdims=True)
    first_pos = np.arange(n_pages) * PAGE + 1
    ms = (rng.random((U, n_pages)) < p_milestone) & (first_pos > P)[None, :]
    ms_strength = (rng.uniform(0.2, 1.0, (U, n_pages)) * ms).astype(np.float32)
    # resident logical pages per unit: prompt 0..Pp-1, m_cur, and nd - 1 of [m_cur - span*nd, m_cur)
    cand = np.arange(m_cur - span * nd, m_cur)
    logical = np.zeros((U, C), np.int64)
    logical[:, :Pp] = np.arange(Pp)
    pick_score = ms_strength[:, cand] + 0.05 * rng.random((U, len(cand)))
    older = cand[np.argsort(-pick_score, axis=1, kind="stable")[:, : nd - 1]]
    dec = np.concatenate([older, np.full((U, 1), m_cur)], axis=1)
    perm = rng.permuted(np.tile(np.arange(nd), (U, 1)), axis=1)       # random physical slots
    logical[:, Pp:] = np.take_along_axis(dec, perm, axis=1)
    start = (PAGE * logical + 1).astype(np.int32)
    count = np.full((U, C), PAGE, np.int32)
    count[logical == m_cur] = cur_count
    pinned = np.zeros((U, C), np.uint8)
    pinned[:, :Pp] = 1
    last = start + count - 1
    ts = np.minimum(t_now, last + rng.integers(0, 8 * PAGE, (U, C))).astype(np.int32)
    ts[logical == m_cur] = t_now
    ts[:, :Pp] = 0
    state = dict(t=np.full(U, t_now, np.int32), ts=ts, start=start, count=count, pinned=pinned)
    # the stores: row i of a resident page holds position start + i (rows >= count are unused)
    k_st = np.empty((U, C, PAGE, d), np.uint16)
    v_st = np.empty((U, C, PAGE, d), np.uint16)
    for u in range(U):
        z = rng.standard_normal((C, PAGE, d), dtype=np.float32)
        k_st[u] = bf16_bits(phi[u, logical[u]][:, None, :] + key_noise * z / np.sqrt(d))
        v_st[u] = bf16_bits(rng.standard_normal((C, PAGE, d), dtype=np.float32))
    # the next T steps (new token at position t = t_now + 1 + i)
    pp = Pp
    phoenix_until = np.full(U, -1, np.int64)
    phoenix_page = np.zeros(U, np.int64)
    q = np.empty((T, B, Hq, d), np.float32)
    kn = np.empty((T, B, Hkv, d), np.float32)
    for i in range(T):
        t = t_now + 1 + i
        cur = (t - 1) // PAGE
        lo = max(0, cur - int(16 * milestone_half_life / PAGE))      # older milestones: < 2^-16
        age = t - first_pos[lo: cur + 1]
        w = ms_strength[:, lo: cur + 1] * (2.0 ** (-np.maximum(age, 0) / milestone_half_life))[None, :]
        w[:, cur - lo] = np.maximum(w[:, cur - lo], recent_weight)
        w[:, cur - 1 - lo] = np.maximum(w[:, cur - 1 - lo], recent_weight)
        start_ph = (rng.random(U) < p_phoenix) & (phoenix_until < t)
        phoenix_page[start_ph] = rng.integers(0, pp, int(start_ph.sum()))
        phoenix_until[start_ph] = t + phoenix_len
        base = np.einsum("up,upd->ud", w, phi[:, lo: cur + 1])
        base += phi[:, 0]                                             # sink ("lazy" maps)
        act = (phoenix_until >= t) & (phoenix_page != 0)              # page 0 is the sink already
        base[act] += phoenix_weight * phi[act, phoenix_page[act]]
        base *= lam * np.sqrt(d)
        noise = eta * rng.standard_normal((U, g, d), dtype=np.float32)
        q[i] = (base[:, None, :] + noise).reshape(B, Hq, d)
        kn[i] = (phi[:, cur] + key_noise * rng.standard_normal((U, d), dtype=np.float32) / np.sqrt(d)
                 ).reshape(B, Hkv, d)
    vn = rng.standard_normal((T, B, Hkv, d), dtype=np.float32)
    steps = Stream(None, None, bf16_bits(q), bf16_bits(kn), bf16_bits(vn))
    return state, k_st, v_st, steps
