"""Pins for the CPU oracle: each check is fixed by the paper or
by mathematics, never by the oracle itself.  CPU only."""
import itertools
import math

import numpy as np
import pytest

from paper_2502_11147_b200.synth import bf16_to_f32, gaussian_stream, waterfall_stream
from traces import hand_trace_stream, page_twin_stream

PAGE = 16


def run_oracle(oracle_mod, stream, L, alpha, page, Hq, Hkv, on_step=None):
    B, _, P, d = stream.k_pre.shape
    o = oracle_mod.Oracle(L=L, alpha=alpha, page=page, n_q_heads=Hq, n_kv_heads=Hkv,
                          head_dim=d, batch=B)
    o.prefill(stream.k_pre, stream.v_pre, P)
    outs = []
    for i in range(stream.T):
        out = o.decode_step(stream.q[i], stream.k[i], stream.v[i])
        outs.append(out)
        if on_step is not None:
            on_step(i, P + i + 1, o, out)
    return o, outs


def positions_kv(stream):
    """K, V for every position 1..P+T as fp64 arrays [B, Hkv, N, d] (index pos-1)."""
    K = np.concatenate([bf16_to_f32(stream.k_pre), np.moveaxis(bf16_to_f32(stream.k), 0, 2)], axis=2)
    V = np.concatenate([bf16_to_f32(stream.v_pre), np.moveaxis(bf16_to_f32(stream.v), 0, 2)], axis=2)
    return K.astype(np.float64), V.astype(np.float64)


def textbook_attention(q, K, V, scale):
    """softmax(scale * q K^T) V for one head, fp64 (Vaswani et al.; PAPER.md :70)."""
    s = scale * (K @ q)
    w = np.exp(s - s.max())
    w /= w.sum()
    return w @ V


# ---------------------------------------------------------------- P3 hand trace


def test_p3_hand_trace_token_level(oracle_mod):
    g, st = hand_trace_stream()
    s, exp = g["setup"], g["expected"]
    evictions = []

    def on_step(i, t, o, out):
        ev = o.get_trace()["evicted"][0]
        if ev >= 0:
            evictions.append([t, int(ev)])

    o, _ = run_oracle(oracle_mod, st, L=s["L"], alpha=s["alpha"], page=1, Hq=1, Hkv=1,
                      on_step=on_step)
    assert evictions == exp["evictions"]
    assert o.resident_positions(0).tolist() == exp["final_resident"]
    state = o.get_state()
    ts_by_pos = {int(p): int(t) for p, t, pin in zip(state["start"][0], state["ts"][0], state["pinned"][0]) if not pin}
    assert ts_by_pos == {int(k): v for k, v in exp["final_ts"].items()}


def test_p3_fig5_narrative_facts(oracle_mod):
    """The three facts PAPER.md :100 narrates, read off the same trace."""
    g, st = hand_trace_stream()
    s = g["setup"]
    seen = {}

    def on_step(i, t, o, out):
        state = o.get_state()
        seen[t] = {int(p): int(ts) for p, ts in zip(state["start"][0], state["ts"][0])}
        seen[(t, "ev")] = int(o.get_trace()["evicted"][0])

    run_oracle(oracle_mod, st, L=s["L"], alpha=s["alpha"], page=1, Hq=1, Hkv=1, on_step=on_step)
    # token 4 is attended at t=5 but below alpha: not refreshed (Fig 5 row 4 analogue)
    assert seen[5][4] == 4
    # token 4 exceeds alpha at t=6: it gets the latest timestamp (Fig 5 row 5: "timestamp 5")
    assert seen[6][4] == 6
    # first full step evicts the oldest token (Fig 5 row 6) and the new token is resident
    assert seen[(7, "ev")] == 3 and seen[7].get(7) == 7


def test_p3_page_twin(oracle_mod):
    for gh in (1, 4):
        g, st = page_twin_stream(g_heads=gh, value_seed=3)
        s, exp = g["setup"], g["expected"]
        evictions = []

        def on_step(i, t, o, out):
            ev = o.get_trace()["evicted"][0]
            if ev >= 0:
                evictions.append([t, (int(ev) - 1) // PAGE + 1])

        o, _ = run_oracle(oracle_mod, st, L=s["L"], alpha=s["alpha"], page=PAGE, Hq=gh, Hkv=1,
                          on_step=on_step)
        assert evictions == exp["page_evictions"]
        state = o.get_state()
        pages = sorted((int(sp) - 1) // PAGE + 1 for sp in state["start"][0])
        assert pages == exp["final_pages"]
        ts = {(int(sp) - 1) // PAGE + 1: int(t) for sp, t, pin in
              zip(state["start"][0], state["ts"][0], state["pinned"][0]) if not pin}
        assert ts == {int(k): v for k, v in exp["final_ts"].items()}


# ---------------------------------------------------------------- P1 dense equivalence


@pytest.mark.parametrize("kind,g,d,P", [("gauss", 4, 64, 37), ("water", 2, 64, 32), ("gauss", 1, 32, 5),
                                        ("gauss", 7, 128, 16)])
def test_p1_dense_equivalence(oracle_mod, kind, g, d, P):
    """L >= P+T: nothing is evicted, so every step is textbook causal attention over all
    tokens so far (§2.1 :46-48, :70)."""
    B, Hkv, T = 2, 2, 40
    Hq = g * Hkv
    mk = gaussian_stream if kind == "gauss" else waterfall_stream
    st = mk(11, B, Hq, Hkv, d, P, T)
    L = ((P + T + PAGE - 1) // PAGE + 1) * PAGE
    K, V = positions_kv(st)
    scale = 1.0 / math.sqrt(d)
    maxerr = 0.0

    def on_step(i, t, o, out):
        nonlocal maxerr
        assert (o.get_trace()["evicted"] == -1).all()
        q = bf16_to_f32(st.q[i]).astype(np.float64)
        for b in range(B):
            for h in range(Hq):
                kv = h // g
                ref = textbook_attention(q[b, h], K[b, kv, :t], V[b, kv, :t], scale)
                maxerr = max(maxerr, np.abs(ref - out[b, h]).max())

    run_oracle(oracle_mod, st, L=L, alpha=1e-4, page=PAGE, Hq=Hq, Hkv=Hkv, on_step=on_step)
    assert maxerr < 1e-12


# ---------------------------------------------------------------- P2 invariants + P8


def test_p2_invariants_and_p8_resident_attention(oracle_mod):
    """Every step: prefill resident, occupancy <= L, ts <= t, ts >= last write, pages hold
    consecutive positions, evicted positions never return (no recall, D19), and `out`
    equals textbook attention over exactly the resident positions (P8)."""
    B, Hkv, g, d, P, T, L = 2, 2, 4, 64, 40, 300, 128
    Hq = g * Hkv
    st = waterfall_stream(5, B, Hq, Hkv, d, P, T, lam=6.0)
    K, V = positions_kv(st)
    scale = 1.0 / math.sqrt(d)
    gone = [set() for _ in range(B * Hkv)]
    prev = [None] * (B * Hkv)
    n_ev = 0
    stamped = []

    def on_step(i, t, o, out):
        nonlocal n_ev
        state = o.get_state()
        tr = o.get_trace()
        q = bf16_to_f32(st.q[i]).astype(np.float64)
        for u in range(B * Hkv):
            res = o.resident_positions(u)
            rs = set(res.tolist())
            assert set(range(1, P + 1)) <= rs                     # prefill pinned (:396)
            assert len(res) <= L                                   # O(L) memory (:191-193)
            assert t in rs                                         # new token attended (D20)
            assert len(rs) == len(res)
            if prev[u] is not None:
                gone[u] |= prev[u] - rs
            assert not (gone[u] & rs)                              # no recall (D19)
            prev[u] = rs
            for p in range(o.C):
                c, s0, ts, pin = (state["count"][u, p], state["start"][u, p], state["ts"][u, p],
                                  state["pinned"][u, p])
                if c == 0:
                    continue
                assert s0 + c - 1 <= t
                if not pin:
                    assert s0 + c - 1 <= ts <= t                   # ts >= last write (D8), <= now
                    stamped.append(ts == t)
            if tr["evicted"][u] >= 0:
                n_ev += 1
            b, kv = divmod(u, Hkv)
            idx = res - 1
            for j in range(g):
                h = kv * g + j
                ref = textbook_attention(q[b, h], K[b, kv, idx], V[b, kv, idx], scale)
                assert np.abs(ref - out[b, h]).max() < 1e-12

    run_oracle(oracle_mod, st, L=L, alpha=1e-4, page=PAGE, Hq=Hq, Hkv=Hkv, on_step=on_step)
    assert n_ev > 0
    rate = np.mean(stamped)
    assert 0.05 < rate < 0.95, rate                                # waterfall data is selective


# ---------------------------------------------------------------- P4 alpha in {0, >=1}


def sliding_window(P, L, t, page=PAGE):
    """StreamingLLM at page granularity (PAPER.md :70, :223): pinned prefill pages plus
    the most recent C-Pp decode pages."""
    C, Pp = L // page, -(-P // page)
    B0 = Pp * page
    if t <= B0:
        return list(range(1, t + 1))
    kc = (t - B0 - 1) // page
    res = list(range(1, B0 + 1))
    for k in range(max(0, kc - (C - Pp) + 1), kc + 1):
        res += list(range(B0 + page * k + 1, min(B0 + page * k + page, t) + 1))
    return res


@pytest.mark.parametrize("P,L,T", [(32, 64, 256), (100, 128, 300), (20, 48, 100), (0, 32, 80)])
@pytest.mark.parametrize("alpha", [0.0, 1.0, 3.0])
def test_p4_alpha_extremes_are_sliding_window(oracle_mod, P, L, T, alpha):
    st = gaussian_stream(7, 1, 2, 1, 16, P, T)

    def on_step(i, t, o, out):
        assert o.resident_positions(0).tolist() == sliding_window(P, L, t)
        state = o.get_state()
        unp = (state["pinned"][0] == 0) & (state["count"][0] > 0)
        if alpha == 0.0:                       # ln 0 = -inf: every page stamped every step
            assert (state["ts"][0][unp] == t).all()
        else:                                  # s - LSE <= 0 <= ln(alpha): nothing stamped
            last = state["start"][0] + state["count"][0] - 1
            assert (state["ts"][0][unp] == last[unp]).all()

    run_oracle(oracle_mod, st, L=L, alpha=alpha, page=PAGE, Hq=2, Hkv=1, on_step=on_step)


# ---------------------------------------------------------------- P5 brute-force bookkeeping


def brute_force_bookkeeping(P, L, page, stamp_steps):
    """Reference recomputed from the full event history (PAPER.md :364, :394, :396):
    a page's timestamp is the latest time it was written or stamped; the victim is the
    unpinned page with the smallest (timestamp, first position).  Slots are filled
    lowest-empty-first.  Returns per-step [(start, count, ts) per slot] and evictions."""
    C, Pp = L // page, -(-P // page)
    slots = [None] * C
    for p in range(Pp):
        pos = list(range(p * page + 1, min(p * page + page, P) + 1))
        slots[p] = dict(pos=pos, events=[], pinned=True)
    t, last_pos = P, P
    hist = []
    for stamps in stamp_steps:
        t += 1
        cur = None
        for s, pg in enumerate(slots):
            if pg is not None and last_pos in pg["pos"]:
                cur = s
        ev = -1
        if cur is not None and len(slots[cur]["pos"]) < page:
            slot = cur
        else:
            empty = [s for s, pg in enumerate(slots) if pg is None]
            if empty:
                slot = empty[0]
            else:
                cands = sorted((max(pg["events"]), pg["pos"][0], s)
                               for s, pg in enumerate(slots) if not pg["pinned"])
                slot = cands[0][2]
                ev = slots[slot]["pos"][0]
            slots[slot] = dict(pos=[], events=[], pinned=False)
        slots[slot]["pos"].append(t)
        slots[slot]["events"].append(t)
        last_pos = t
        for s in stamps:
            if slots[s] is not None and not slots[s]["pinned"]:
                slots[s]["events"].append(t)
        snap = []
        for pg in slots:
            if pg is None:
                snap.append((0, 0, 0))
            else:
                snap.append((pg["pos"][0], len(pg["pos"]), 0 if pg["pinned"] else max(pg["events"])))
        hist.append((snap, ev))
    return hist


@pytest.mark.parametrize("page,P,L,T", [(1, 1, 4, 5), (2, 2, 6, 7), (2, 3, 8, 6), (1, 0, 3, 5)])
def test_p5_bookkeeping_enumeration(oracle_mod, page, P, L, T):
    C, Pp = L // page, -(-P // page)
    dec = list(range(Pp, C))
    nd = len(dec)
    n = 1 << (nd * T)
    o = oracle_mod.Oracle(L=L, alpha=1e-4, page=page, n_q_heads=1, n_kv_heads=1, head_dim=1, batch=n)
    zeros = np.zeros((n, 1, P, 1), np.uint16)
    o.prefill(zeros, zeros, P)
    pats = np.arange(n, dtype=np.int64)
    got = []
    for i in range(T):
        stamps = np.zeros((n, C), np.uint8)
        for j, s in enumerate(dec):
            stamps[:, s] = (pats >> (i * nd + j)) & 1
        o.step_stamps(stamps)
        got.append((o.get_state(), o.get_trace()["evicted"].copy()))
    for u in range(n):
        steps = [[dec[j] for j in range(nd) if (u >> (i * nd + j)) & 1] for i in range(T)]
        ref = brute_force_bookkeeping(P, L, page, steps)
        for i, (snap, ev) in enumerate(ref):
            state, evs = got[i]
            mine = list(zip(state["start"][u].tolist(), state["count"][u].tolist(),
                            np.where(state["pinned"][u] != 0, 0, state["ts"][u]).tolist()))
            assert mine == snap, (u, i)
            assert evs[u] == ev, (u, i)


# ---------------------------------------------------------------- P6 brute-force end-to-end


def brute_force_end_to_end(stream, L, alpha, page, g, scope=0):
    """From-scratch simulator: token positions, direct exp/sum per step (no streaming
    LSE), stamp iff exp(s - LSE) > alpha, evict min (ts, first position).
    scope 0: one page table per (request, kv-head); scope 1: one table per request shared by
    all its kv-heads, stamped if any of its q-heads exceeds alpha (D25).  Returns, per unit
    (request, kv-head), the per-step (state snapshot, evicted position, outputs, margin)."""
    K, V = positions_kv(stream)
    B, Hkv, P, d = stream.k_pre.shape
    C, Pp = L // page, -(-P // page)
    scale = 1.0 / math.sqrt(d)
    tables = [[kv] for kv in range(Hkv)] if scope == 0 else [list(range(Hkv))]
    res = {}
    for b in range(B):
        for kvs in tables:
            pages = []  # dicts: positions, ts, pinned, slot
            for p in range(Pp):
                pages.append(dict(pos=list(range(p * page + 1, min(p * page + page, P) + 1)),
                                  ts=0, pinned=True, slot=p))
            per_step = []
            for i in range(stream.T):
                t = P + i + 1
                cur = max(pages, key=lambda pg: pg["pos"][-1]) if pages else None
                ev = -1
                if cur is not None and len(cur["pos"]) < page:
                    tgt = cur
                else:
                    if len(pages) < C:
                        tgt = dict(pos=[], ts=0, pinned=False, slot=len(pages))
                        pages.append(tgt)
                    else:
                        victim = min((pg for pg in pages if not pg["pinned"]),
                                     key=lambda pg: (pg["ts"], pg["pos"][0]))
                        ev = victim["pos"][0]
                        victim.update(pos=[], pinned=False)
                        tgt = victim
                tgt["pos"].append(t)
                if not tgt["pinned"]:
                    tgt["ts"] = t
                q = bf16_to_f32(stream.q[i, b]).astype(np.float64)
                allpos = sorted(x for pg in pages for x in pg["pos"])
                idx = np.array(allpos) - 1
                outs, probs = {}, []
                for kv in kvs:
                    outs[kv] = []
                    for j in range(g):
                        s = scale * (K[b, kv, idx] @ q[kv * g + j])
                        e = np.exp(s)
                        pr = e / e.sum()
                        outs[kv].append(pr @ V[b, kv, idx])
                        probs.append(dict(zip(allpos, pr)))
                for pg in pages:
                    if not pg["pinned"] and any(pr[x] > alpha for pr in probs for x in pg["pos"]):
                        pg["ts"] = t
                margin = min(abs(pr[x] - alpha) for pr in probs for x in allpos)
                snap = sorted((pg["slot"], pg["pos"][0], len(pg["pos"]), pg["ts"]) for pg in pages)
                per_step.append((snap, ev, {kv: np.array(o) for kv, o in outs.items()}, margin))
            for kv in kvs:
                res[b * Hkv + kv] = [(sn, ev, o[kv], m) for sn, ev, o, m in per_step]
    return [res[u] for u in range(B * Hkv)]


@pytest.mark.parametrize("page,L,P,g,alpha", [(1, 6, 2, 1, 0.12), (2, 6, 2, 2, 0.08), (1, 5, 1, 3, 0.15),
                                              (2, 8, 3, 1, 0.1)])
def test_p6_brute_force_end_to_end(oracle_mod, page, L, P, g, alpha):
    B, Hkv, d, T = 2, 2, 4, 8
    st = gaussian_stream(100 + page * 10 + L, B, g * Hkv, Hkv, d, P, T, sigma_q=2.0)
    ref = brute_force_end_to_end(st, L, alpha, page, g)
    got = []

    def on_step(i, t, o, out):
        got.append((o.get_state(), o.get_trace()["evicted"].copy(), out.copy()))

    run_oracle(oracle_mod, st, L=L, alpha=alpha, page=page, Hq=g * Hkv, Hkv=Hkv, on_step=on_step)
    n_mixed = 0
    for u in range(B * Hkv):
        b, kv = divmod(u, Hkv)
        for i in range(T):
            snap, ev, outs, margin = ref[u][i]
            assert margin > 1e-9, "borderline draw; change the seed"
            state, evs, out = got[i]
            mine = sorted((p, int(state["start"][u, p]), int(state["count"][u, p]),
                           int(state["ts"][u, p])) for p in range(L // page) if state["count"][u, p] > 0)
            assert mine == snap, (u, i)
            assert evs[u] == ev
            assert np.abs(out[b, kv * g:(kv + 1) * g] - outs).max() < 1e-12
            n_mixed += ev >= 0
    assert n_mixed > 0


@pytest.mark.parametrize("page,L,P,Hkv,g,alpha", [(1, 6, 2, 2, 1, 0.12), (2, 6, 2, 3, 2, 0.08),
                                                  (2, 8, 3, 2, 1, 0.1), (1, 5, 1, 4, 1, 0.15)])
def test_request_table_brute_force(oracle_mod, page, L, P, Hkv, g, alpha):
    """table_scope = 1 (D25): one page table per request, stamped by any of its
    q-heads, pinned against the from-scratch simulator; every kv-head holds the same state."""
    B, d, T = 2, 4, 8
    st = gaussian_stream(300 + page * 10 + L + Hkv, B, g * Hkv, Hkv, d, P, T, sigma_q=2.0)
    ref = brute_force_end_to_end(st, L, alpha, page, g, scope=1)
    o = oracle_mod.Oracle(L=L, alpha=alpha, page=page, n_q_heads=g * Hkv, n_kv_heads=Hkv,
                          head_dim=d, batch=B, table_scope=1)
    o.prefill(st.k_pre, st.v_pre, P)
    n_mixed = 0
    for i in range(T):
        out = o.decode_step(st.q[i], st.k[i], st.v[i])
        state, evs = o.get_state(), o.get_trace()["evicted"]
        for u in range(B * Hkv):
            b, kv = divmod(u, Hkv)
            snap, ev, outs, margin = ref[u][i]
            assert margin > 1e-9, "borderline draw; change the seed"
            mine = sorted((p, int(state["start"][u, p]), int(state["count"][u, p]),
                           int(state["ts"][u, p])) for p in range(L // page) if state["count"][u, p] > 0)
            assert mine == snap, (u, i)
            assert evs[u] == ev
            assert np.abs(out[b, kv * g:(kv + 1) * g] - outs).max() < 1e-12
            n_mixed += ev >= 0
        for k in ("ts", "start", "count", "pinned"):   # replicas identical within a request
            a = state[k].reshape(B, Hkv, -1)
            assert (a == a[:, :1]).all()
    assert n_mixed > 0


def test_request_table_differs_from_per_head_tables(oracle_mod):
    """The two granularities are different methods: on a stream whose kv-heads attend
    different pages, per-head tables and the per-request table evict differently."""
    B, Hkv, g, d, P, T, L = 1, 2, 1, 8, 16, 120, 64
    st = gaussian_stream(7, B, g * Hkv, Hkv, d, P, T, sigma_q=3.0)
    ev = []
    for scope in (0, 1):
        o = oracle_mod.Oracle(L=L, alpha=0.02, page=PAGE, n_q_heads=g * Hkv, n_kv_heads=Hkv,
                              head_dim=d, batch=B, table_scope=scope)
        o.prefill(st.k_pre, st.v_pre, P)
        e = []
        for i in range(T):
            o.decode_step(st.q[i], st.k[i], st.v[i], want_out=False)
            e.append(o.get_trace()["evicted"].copy())
        ev.append(np.array(e))
    assert (ev[1][:, 0] == ev[1][:, 1]).all()
    assert not (ev[0][:, 0] == ev[0][:, 1]).all()


# ---------------------------------------------------------------- errors


def test_oracle_error_codes(oracle_mod):
    O = oracle_mod.Oracle
    with pytest.raises(oracle_mod.OracleError):
        O(L=50, alpha=1e-4, page=16, n_q_heads=4, n_kv_heads=2, head_dim=8, batch=1)   # L % page
    with pytest.raises(oracle_mod.OracleError):
        O(L=64, alpha=1e-4, page=16, n_q_heads=3, n_kv_heads=2, head_dim=8, batch=1)   # Hq % Hkv
    o = O(L=64, alpha=1e-4, page=16, n_q_heads=2, n_kv_heads=1, head_dim=8, batch=1)
    z = np.zeros((1, 2, 8), np.uint16)
    with pytest.raises(oracle_mod.OracleError) as e:
        o.decode_step(z, z[:, :1], z[:, :1])                                            # before prefill
    assert e.value.code == oracle_mod.REF_E_STATE
    kp = np.zeros((1, 1, 49, 8), np.uint16)
    with pytest.raises(oracle_mod.OracleError) as e:
        o.prefill(kp, kp, 49)                                                           # D14 budget
    assert e.value.code == oracle_mod.REF_E_BUDGET
    o.prefill(kp[:, :, :48], kp[:, :, :48], 48)
    with pytest.raises(oracle_mod.OracleError) as e:
        o.prefill(kp[:, :, :48], kp[:, :, :48], 48)                                     # twice
    assert e.value.code == oracle_mod.REF_E_STATE


def test_d3_strict_threshold(oracle_mod):
    """D3: "above" alpha (:29), "exceeds" (:100), "exceeding" (:364) -> strict '>'.
    With q = 0 every resident token has p = 1/n exactly; with n = 4 and alpha = 1/4 the
    two unpinned, not-just-written tokens sit exactly on the threshold and must NOT be
    stamped (their timestamps stay at their write times)."""
    d = 8
    o = oracle_mod.Oracle(L=8, alpha=0.25, page=1, n_q_heads=1, n_kv_heads=1, head_dim=d, batch=1)
    rng = np.random.default_rng(0)
    from paper_2502_11147_b200.synth import bf16_bits
    kv = lambda *s: bf16_bits(rng.standard_normal(s).astype(np.float32))
    o.prefill(kv(1, 1, 1, d), kv(1, 1, 1, d), 1)
    zero_q = np.zeros((1, 1, d), np.uint16)
    for _ in range(3):                      # t = 2, 3, 4
        o.decode_step(zero_q, kv(1, 1, d), kv(1, 1, d))
    st = o.get_state()
    ts = {int(s): int(t) for s, t, c in zip(st["start"][0], st["ts"][0], st["count"][0]) if c}
    assert ts == {1: 0, 2: 3, 3: 3, 4: 4}    # t=3: p=1/3 > 1/4 stamps 2; t=4: p=1/4 stamps nothing
    o.close()
    o = oracle_mod.Oracle(L=8, alpha=0.2499, page=1, n_q_heads=1, n_kv_heads=1, head_dim=d, batch=1)
    o.prefill(kv(1, 1, 1, d), kv(1, 1, 1, d), 1)
    for _ in range(3):
        o.decode_step(zero_q, kv(1, 1, d), kv(1, 1, d))
    st = o.get_state()
    ts = {int(s): int(t) for s, t, c in zip(st["start"][0], st["ts"][0], st["count"][0]) if c}
    assert ts == {1: 0, 2: 4, 3: 4, 4: 4}


# ---------------------------------------------------------------- NEXT-1: Quest bound mode


def _dense_pstars(oracle_mod, st, g, score_mode, page=PAGE):
    B, Hkv, P, d = st.k_pre.shape
    L = ((P + st.T) // page + 2) * page
    o = oracle_mod.Oracle(L=L, alpha=1e-4, page=page, n_q_heads=g * Hkv, n_kv_heads=Hkv,
                          head_dim=d, batch=B, score_mode=score_mode)
    o.prefill(st.k_pre, st.v_pre, P)
    out = []
    for i in range(st.T):
        o.decode_step(st.q[i], st.k[i], st.v[i])
        out.append(o.get_trace()["pstar"].copy())
    return np.stack(out)


def test_quest_bound_dominates_exact_page_max(oracle_mod):
    """Quest's per-channel min/max bound (PAPER.md :147-151, :362) is an upper bound of every
    token's logit in the page, so with identical residency (L >= N: no eviction) its estimated
    score is >= the exact page max everywhere, and its stamp set is a superset."""
    st = waterfall_stream(17, 2, 8, 2, 64, 40, 60)
    ex = _dense_pstars(oracle_mod, st, 4, 0)
    qu = _dense_pstars(oracle_mod, st, 4, 1)
    valid = ex >= 0
    assert valid.any()
    assert (qu[valid] >= ex[valid] * (1 - 1e-12)).all()
    assert ((qu > 1e-4) | ~(ex > 1e-4)).all()          # stamps(quest) ⊇ stamps(exact)
    assert (qu[valid] > ex[valid] * (1 + 1e-9)).any()  # and strictly looser somewhere


def test_quest_bound_is_exact_for_single_token_pages(oracle_mod):
    """page = 1: the representative key IS the key, so both modes give the same scores."""
    st = gaussian_stream(18, 2, 4, 2, 16, 5, 30)
    ex = _dense_pstars(oracle_mod, st, 2, 0, page=1)
    qu = _dense_pstars(oracle_mod, st, 2, 1, page=1)
    assert np.allclose(qu, ex, rtol=1e-12, atol=0)


def test_quest_bound_is_exact_for_identical_keys(oracle_mod):
    """All keys of a page equal: min = max = k, so U = q.k exactly (P3' page twin data)."""
    g_, st = page_twin_stream(g_heads=2, value_seed=1)
    st.T  # noqa: B018
    short = type(st)(st.k_pre, st.v_pre, st.q[:40], st.k[:40], st.v[:40])
    ex = _dense_pstars(oracle_mod, short, 2, 0)
    qu = _dense_pstars(oracle_mod, short, 2, 1)
    assert np.allclose(qu, ex, rtol=1e-12, atol=0)


# ---------------------------------------------------------------- NEXT-2: variable prompts


def test_varlen_prefill_equals_independent_requests(oracle_mod):
    """Requests with different prompt lengths in one batch behave exactly like separate
    single-request runs (units are independent, reading D5): same state, same outputs."""
    B, Hq, Hkv, d, Pmax, T, L = 3, 8, 2, 32, 50, 120, 96
    Ps = [50, 17, 0]
    st = waterfall_stream(23, B, Hq, Hkv, d, Pmax, T)
    o = oracle_mod.Oracle(L=L, alpha=1e-4, page=PAGE, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, batch=B)
    o.prefill_varlen(st.k_pre, st.v_pre, Ps)
    singles = []
    for b, P in enumerate(Ps):
        s1 = oracle_mod.Oracle(L=L, alpha=1e-4, page=PAGE, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, batch=1)
        s1.prefill(np.ascontiguousarray(st.k_pre[b:b + 1, :, :P]), np.ascontiguousarray(st.v_pre[b:b + 1, :, :P]), P)
        singles.append(s1)
    for i in range(T):
        out = o.decode_step(st.q[i], st.k[i], st.v[i])
        stv = o.get_state()
        for b, s1 in enumerate(singles):
            o1 = s1.decode_step(st.q[i][b:b + 1], st.k[i][b:b + 1], st.v[i][b:b + 1])
            assert np.array_equal(out[b:b + 1], o1)
            s1s = s1.get_state()
            for k in ("t", "ts", "start", "count", "pinned"):
                assert np.array_equal(stv[k][b * Hkv:(b + 1) * Hkv], s1s[k])
    assert o.get_state()["t"].tolist() == [P + T for P in Ps for _ in range(Hkv)]


# ---------------------------------------------------------------- NEXT-3: top-r stamping


@pytest.mark.parametrize("r,closed", [(1.0, "alpha0"), (0.0, "alpha1")])
def test_top_r_extremes_are_sliding_window(oracle_mod, r, closed):
    """r = 1 stamps every decision page (= alpha 0), r = 0 none (= alpha >= 1): both reduce to
    the StreamingLLM window of P4."""
    P, L, T = 100, 128, 300
    st = gaussian_stream(7, 1, 2, 1, 16, P, T)
    o = oracle_mod.Oracle(L=L, alpha=0.5, page=PAGE, n_q_heads=2, n_kv_heads=1, head_dim=16,
                          batch=1, stamp_rule=1, top_r=r)
    o.prefill(st.k_pre, st.v_pre, P)
    for i in range(T):
        o.decode_step(st.q[i], st.k[i], st.v[i])
        assert o.resident_positions(0).tolist() == sliding_window(P, L, P + i + 1)


def brute_force_top_r(stream, L, r, page, g):
    """From-scratch simulator of the top-r rule (PAPER.md :135, reading D23): each step, stamp
    the ceil(r n) unpinned resident pages with the largest max-probability (ties to the oldest
    page), direct exp/sum per step."""
    K, V = positions_kv(stream)
    B, Hkv, P, d = stream.k_pre.shape
    C, Pp = L // page, -(-P // page)
    scale = 1.0 / math.sqrt(d)
    res = []
    for b in range(B):
        for kv in range(Hkv):
            pages = [dict(pos=list(range(p * page + 1, min(p * page + page, P) + 1)), ts=0,
                          pinned=True, slot=p) for p in range(Pp)]
            per_step = []
            for i in range(stream.T):
                t = P + i + 1
                cur = max(pages, key=lambda pg: pg["pos"][-1]) if pages else None
                if cur is not None and len(cur["pos"]) < page:
                    tgt = cur
                elif len(pages) < C:
                    tgt = dict(pos=[], ts=0, pinned=False, slot=len(pages))
                    pages.append(tgt)
                else:
                    tgt = min((pg for pg in pages if not pg["pinned"]), key=lambda pg: (pg["ts"], pg["pos"][0]))
                    tgt.update(pos=[], pinned=False)
                tgt["pos"].append(t)
                if not tgt["pinned"]:
                    tgt["ts"] = t
                q = bf16_to_f32(stream.q[i, b]).astype(np.float64)
                allpos = sorted(x for pg in pages for x in pg["pos"])
                idx = np.array(allpos) - 1
                probs = []
                for j in range(g):
                    e = np.exp(scale * (K[b, kv, idx] @ q[kv * g + j]))
                    probs.append(dict(zip(allpos, e / e.sum())))
                dec = [pg for pg in pages if not pg["pinned"]]
                score = {id(pg): max(pr[x] for pr in probs for x in pg["pos"]) for pg in dec}
                k = int(np.ceil(np.float32(r) * np.float32(len(dec))))
                ranked = sorted(dec, key=lambda pg: (-score[id(pg)], pg["pos"][0]))
                for pg in ranked[:k]:
                    pg["ts"] = t
                per_step.append(sorted((pg["slot"], pg["pos"][0], len(pg["pos"]), pg["ts"]) for pg in pages))
            res.append(per_step)
    return res


@pytest.mark.parametrize("page,L,P,g,r", [(1, 6, 2, 1, 0.5), (2, 8, 2, 2, 0.5), (2, 10, 3, 1, 0.3),
                                          (1, 7, 1, 3, 0.25)])
def test_top_r_brute_force(oracle_mod, page, L, P, g, r):
    B, Hkv, d, T = 2, 2, 4, 10
    st = gaussian_stream(200 + L + P, B, g * Hkv, Hkv, d, P, T, sigma_q=2.0)
    ref = brute_force_top_r(st, L, r, page, g)
    o = oracle_mod.Oracle(L=L, alpha=1e-4, page=page, n_q_heads=g * Hkv, n_kv_heads=Hkv,
                          head_dim=d, batch=B, stamp_rule=1, top_r=r)
    o.prefill(st.k_pre, st.v_pre, P)
    for i in range(T):
        o.decode_step(st.q[i], st.k[i], st.v[i])
        state = o.get_state()
        for u in range(B * Hkv):
            mine = sorted((p, int(state["start"][u, p]), int(state["count"][u, p]),
                           int(state["ts"][u, p])) for p in range(L // page) if state["count"][u, p] > 0)
            assert mine == ref[u][i], (u, i)


# ---------------------------------------------------------------- NEXT-4: Quest-on-prefill hybrid


def _hybrid_stream(seed, B=2, Hkv=2, g=2, d=32, n_prompt_pages=8, T=90):
    """Prompt pages whose 16 keys are identical (so Quest's bound equals the exact logit),
    random decode keys, random values and queries."""
    rng = np.random.default_rng(seed)
    from paper_2502_11147_b200.synth import Stream, bf16_bits
    P = PAGE * n_prompt_pages
    phi = rng.standard_normal((B, Hkv, n_prompt_pages, d)) * 0.7
    k_pre = np.repeat(phi, PAGE, axis=2).astype(np.float32)
    v_pre = rng.standard_normal((B, Hkv, P, d)).astype(np.float32)
    q = rng.standard_normal((T, B, Hkv * g, d)).astype(np.float32) * 1.5
    k = rng.standard_normal((T, B, Hkv, d)).astype(np.float32) * 0.5
    v = rng.standard_normal((T, B, Hkv, d)).astype(np.float32)
    return Stream(bf16_bits(k_pre), bf16_bits(v_pre), bf16_bits(q), bf16_bits(k), bf16_bits(v))


def test_hybrid_selects_top_k_prompt_pages_and_attends_exactly_those(oracle_mod):
    """Quest on the prompt + RaaS on decode (PAPER.md :173/:183, :237; reading D24).  With
    constant keys inside each prompt page the bound is the exact logit, so the selection is
    the K pages with the largest max_h q_h.phi_p, and out is textbook attention over the
    selected prompt pages plus the resident decode tokens."""
    B, Hkv, g, d, npp, T, K = 2, 2, 2, 32, 8, 90, 3
    st = _hybrid_stream(3, B, Hkv, g, d, npp, T)
    P, L = PAGE * npp, PAGE * npp + 64
    o = oracle_mod.Oracle(L=L, alpha=1e-4, page=PAGE, n_q_heads=Hkv * g, n_kv_heads=Hkv, head_dim=d,
                          batch=B, quest_prefill_pages=K)
    o.prefill(st.k_pre, st.v_pre, P)
    Kp, Vp = positions_kv(st)
    scale = 1.0 / math.sqrt(d)
    phi = bf16_to_f32(st.k_pre)[:, :, ::PAGE].astype(np.float64)     # [B, Hkv, npp, d]
    for i in range(T):
        out = o.decode_step(st.q[i], st.k[i], st.v[i])
        sel = o.get_selection()
        q = bf16_to_f32(st.q[i]).astype(np.float64)
        for b in range(B):
            for kv in range(Hkv):
                u = b * Hkv + kv
                sc = np.max(np.einsum("hd,pd->hp", q[b, kv * g:(kv + 1) * g], phi[b, kv]), axis=0)
                top = sorted(np.argsort(-sc, kind="stable")[:K].tolist())
                assert np.flatnonzero(sel["attended"][u, :npp]).tolist() == top
                res = o.resident_positions(u)
                att = [x for x in res if x > P or (x - 1) // PAGE in top]
                idx = np.array(att) - 1
                for j in range(g):
                    ref = textbook_attention(q[b, kv * g + j], Kp[b, kv, idx], Vp[b, kv, idx], scale)
                    assert np.abs(ref - out[b, kv * g + j]).max() < 1e-12


def test_hybrid_with_k_at_least_prompt_pages_is_plain_raas(oracle_mod):
    st = _hybrid_stream(4)
    P, L = PAGE * 8, PAGE * 8 + 64
    outs, states = [], []
    for K in (0, 8, 20):
        o = oracle_mod.Oracle(L=L, alpha=1e-4, page=PAGE, n_q_heads=4, n_kv_heads=2, head_dim=32,
                              batch=2, quest_prefill_pages=K)
        o.prefill(st.k_pre, st.v_pre, P)
        outs.append(np.stack([o.decode_step(st.q[i], st.k[i], st.v[i]) for i in range(st.T)]))
        states.append(o.get_state())
    for x in outs[1:]:
        assert np.array_equal(x, outs[0])
    for s_ in states[1:]:
        assert all(np.array_equal(s_[k], states[0][k]) for k in s_)


def test_bench_waterfall_generator_is_selective(oracle_mod):
    """The bench's device-side generator (synth.WaterfallTorch, drawn here on the CPU) keeps
    the waterfall structure of DESIGN.md §4: keys of one logical page share a signature, and
    the page stamp rate is selective (not the ~100 % of i.i.d. data), so eviction is not FIFO."""
    import torch

    from paper_2502_11147_b200.synth import WaterfallTorch

    B, Hq, Hkv, d, P, T, L = 1, 8, 2, 64, 40, 300, 128
    wf = WaterfallTorch(11, B, Hq, Hkv, d, P, T, "cpu", lam=7.0)
    k, v = wf.prefill()
    kf = k.float()[0, 0]
    cos = torch.nn.functional.cosine_similarity(kf[:16, None], kf[None, :16], dim=-1)
    other = torch.nn.functional.cosine_similarity(kf[:16, None], kf[None, 16:32], dim=-1)
    assert cos.mean() > 0.6 and other.abs().mean() < 0.3          # page-correlated keys

    def bits(x):
        return x.contiguous().view(torch.int16).numpy().view(np.uint16)

    o = oracle_mod.Oracle(L=L, alpha=1e-4, page=PAGE, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d,
                          batch=B)
    o.prefill(bits(k), bits(v), P)
    q = torch.empty(B, Hq, d, dtype=torch.bfloat16)
    kn = torch.empty(B, Hkv, d, dtype=torch.bfloat16)
    vn = torch.empty_like(kn)
    stamped, n_ev = [], 0
    for i in range(T):
        wf.step(q, kn, vn)
        o.decode_step(bits(q), bits(kn), bits(vn), want_out=False)
        tr, s = o.get_trace(), o.get_state()
        m = (s["pinned"] == 0) & (s["count"] > 0)
        stamped.extend((tr["pstar"][m] > 1e-4).tolist())
        n_ev += int((tr["evicted"] >= 0).sum())
    rate = float(np.mean(stamped))
    assert n_ev > 0
    assert 0.05 < rate < 0.95, rate


# ---------------------------------------------------------------- resync: set_state(get_state)


def _roundtrip_case(oracle_mod, st, n1, check_split, **cfg):
    """Run the oracle n1 steps, read its whole state (metadata + K/V stores), set it into a FRESH
    oracle and continue both for the rest of the stream: states, stores and outputs must stay
    bitwise identical (the lockstep resync of SURVEY §8c parity protocol rests on this).
    `check_split(state)` asserts the property of the split point the case is about."""
    B, _, P, d = st.k_pre.shape
    a = oracle_mod.Oracle(head_dim=d, batch=B, **cfg)
    a.prefill(st.k_pre, st.v_pre, P)
    for i in range(n1):
        a.decode_step(st.q[i], st.k[i], st.v[i])
    s = a.get_state()
    check_split(s)
    ks, vs = a.get_kv()
    b = oracle_mod.Oracle(head_dim=d, batch=B, **cfg)
    b.set_state(s["t"], s["ts"], s["start"], s["count"], s["pinned"], ks, vs)
    s_b = b.get_state()
    for k in s:
        assert np.array_equal(s[k], s_b[k]), k
    evictions = 0
    for i in range(n1, st.T):
        oa = a.decode_step(st.q[i], st.k[i], st.v[i])
        ob = b.decode_step(st.q[i], st.k[i], st.v[i])
        assert np.array_equal(oa, ob), f"out differs at step {i}"
        sa, sb = a.get_state(), b.get_state()
        for k in sa:
            assert np.array_equal(sa[k], sb[k]), f"state '{k}' differs at step {i}"
        evictions += int((a.get_trace()["evicted"] >= 0).sum())
    ka, va = a.get_kv()
    kb, vb = b.get_kv()
    assert np.array_equal(ka, kb) and np.array_equal(va, vb)
    return evictions


def _cur_page(s, u):
    """the write page: the used page with the largest start position (the page of token t)"""
    used = np.nonzero(s["count"][u] > 0)[0]
    return used[np.argmax(s["start"][u][used])]


@pytest.mark.parametrize("P,n1,where", [
    (40, 3, "partial prompt page"),       # 40 % 16 = 8: decode tokens 41.. fill the pinned page 2
    (40, 157, "partial decode page"),     # after evictions, cur = a victim page being refilled
    (32, 160, "full page"),               # (32 + 160) % 16 == 0: the next step opens a page
])
def test_set_state_roundtrip_continues_bitwise(oracle_mod, P, n1, where):
    """raas_ref_set_state re-derives the write cursor (the used page with the largest start
    position), the used count and the pinned set from the metadata alone.  From a state whose
    current page is partial (prompt or decode) or full, the resynced oracle must continue
    exactly as the uninterrupted one (App. B :394-396: time, prompt pinning, eviction
    of the earliest recorded time)."""
    st = waterfall_stream(4100 + P + n1, 2, 8, 2, 64, P, 260)
    cfg = dict(L=128, alpha=1e-4, page=PAGE, n_q_heads=8, n_kv_heads=2)

    def check(s):
        for u in range(4):
            cur = _cur_page(s, u)
            full = s["count"][u, cur] == PAGE
            if where == "full page":
                assert full
            else:
                assert not full
                assert bool(s["pinned"][u, cur]) == (where == "partial prompt page")
        if P % PAGE:
            assert (s["pinned"][:, P // PAGE] == 2).all() and (s["pinned"][:, : P // PAGE] == 1).all()

    assert _roundtrip_case(oracle_mod, st, n1, check, **cfg) > 0


def test_set_state_roundtrip_token_level(oracle_mod):
    """page = 1 (§3.2): every token its own entry; resync mid-stream after evictions."""
    st = waterfall_stream(4200, 1, 4, 2, 64, 20, 200)
    cfg = dict(L=64, alpha=1e-3, page=1, n_q_heads=4, n_kv_heads=2)
    assert _roundtrip_case(oracle_mod, st, 77, lambda s: None, **cfg) > 0


@pytest.mark.parametrize("n1", [5, 40])
def test_set_state_roundtrip_hybrid_partial_prompt_page(oracle_mod, n1):
    """Quest-on-prefill hybrid (D24) with P % 16 != 0: the prompt's partial last page is flagged
    2 by get_state, never selectable, and always attended -- also after it has been filled by
    decode tokens (n1 = 40) -- so the resynced run attends the same pages.  Taking every pinned
    page as selectable, or none, changes the attended set and therefore out."""
    P, K = 200, 4            # 12 full prompt pages + 8 prompt tokens in page 12
    st = waterfall_stream(4300 + n1, 2, 8, 2, 64, P, 100, p_phoenix=1.0 / 16, phoenix_len=8)
    cfg = dict(L=320, alpha=1e-4, page=PAGE, n_q_heads=8, n_kv_heads=2, quest_prefill_pages=K)

    def check(s):
        assert (s["pinned"][:, :12] == 1).all() and (s["pinned"][:, 12] == 2).all()
        assert (s["count"][:, 12] == (PAGE if n1 >= 8 else 8 + n1)).all()

    _roundtrip_case(oracle_mod, st, n1, check, **cfg)


def test_set_state_roundtrip_request_table_top_r(oracle_mod):
    """One table per request (D25) with the top-r rule (D23): the replicas resync as one."""
    st = waterfall_stream(4400, 2, 8, 2, 64, 24, 220)
    cfg = dict(L=96, alpha=1e-4, page=PAGE, n_q_heads=8, n_kv_heads=2, stamp_rule=1, top_r=0.5,
               table_scope=1)
    assert _roundtrip_case(oracle_mod, st, 101, lambda s: None, **cfg) > 0


def test_set_state_hybrid_flags_select_the_full_prompt_pages(oracle_mod):
    """The pinned flags are what set_state derives the hybrid's selectable pages from: a state
    read from an uninterrupted run but with the partial page re-flagged 1 (i.e. 'every pinned
    page is a full prompt page') must NOT continue like the original -- the check above would be
    vacuous otherwise."""
    P, K = 200, 4
    st = waterfall_stream(4340, 2, 8, 2, 64, P, 100, p_phoenix=1.0 / 16, phoenix_len=8)
    cfg = dict(L=320, alpha=1e-4, page=PAGE, n_q_heads=8, n_kv_heads=2, quest_prefill_pages=K)
    a = oracle_mod.Oracle(head_dim=64, batch=2, **cfg)
    a.prefill(st.k_pre, st.v_pre, P)
    for i in range(40):
        a.decode_step(st.q[i], st.k[i], st.v[i])
    s = a.get_state()
    ks, vs = a.get_kv()
    b = oracle_mod.Oracle(head_dim=64, batch=2, **cfg)
    bad = dict(s, pinned=np.where(s["pinned"] == 2, 1, s["pinned"]).astype(np.uint8))
    b.set_state(bad["t"], bad["ts"], bad["start"], bad["count"], bad["pinned"], ks, vs)
    differs = False
    for i in range(40, st.T):
        oa = a.decode_step(st.q[i], st.k[i], st.v[i])
        ob = b.decode_step(st.q[i], st.k[i], st.v[i])
        differs |= not np.array_equal(oa, ob)
    assert differs
