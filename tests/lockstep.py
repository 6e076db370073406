"""GPU (libraas) vs CPU oracle lockstep driver (SURVEY.md §8c parity protocol).

After every step: metadata (t, ts, start_pos, count, pinned) must be bit-exact; a differing
timestamp is tolerated only when the oracle's decisive probability p* of that page lies within
|p* - alpha| < 1e-6 (a "band event": counted, then the GPU is resynced to the oracle state).
Outputs are compared against the oracle's fp64 result with max abs error <= 2e-2.
"""
import numpy as np
import torch

from paper_2502_11147_b200.raas import RaasLayer
from paper_2502_11147_b200.synth import bf16_to_f32

BAND = 1e-6
OUT_TOL = 2e-2


def to_dev(bits, device="cuda"):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(device)


def from_dev(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


class LockstepResult:
    def __init__(self):
        self.steps = 0
        self.band_events = 0
        self.max_err = 0.0
        self.evictions = 0
        self.stamp_decisions = 0
        self.stamps = 0
        self.gpu_evictions = []   # per step, list of (unit, evicted start_pos)


def _topr_band(pstar_u, p, top_r):
    """top-r rule: a differing decision is allowed only at the k-th boundary (the page's score
    within 1e-6 relative of the oracle's k-th largest score)."""
    dec = np.sort(pstar_u[pstar_u >= 0])[::-1]
    k = int(np.ceil(np.float32(top_r) * np.float32(len(dec))))
    if k == 0 or k > len(dec):
        return False
    kth = dec[k - 1]
    return abs(pstar_u[p] - kth) <= 1e-6 * kth


def compare_state(g, o, alpha, pstar, res, layer, resync=True, top_r=None, history=None):
    """history: pstar of the steps since the last comparison (index -1 = this step), for state
    read back every few steps: a differing timestamp tau is judged by the p* of step tau."""
    keys = ("t", "ts", "start", "count", "pinned")
    same = all(np.array_equal(g[k], o[k]) for k in keys)
    if same:
        return
    # only ts may differ, and only inside the band
    for k in ("t", "start", "count", "pinned"):
        assert np.array_equal(g[k], o[k]), f"state field {k} differs outside the stamp band"
    diff = np.argwhere(g["ts"] != o["ts"])
    for u, p in diff:
        ps = pstar[u, p]
        if history is not None:
            tau = max(int(g["ts"][u, p]), int(o["ts"][u, p]))   # the later stamp is the disputed one
            back = int(o["t"][u]) - tau
            if 0 <= back < len(history):
                ps = history[-1 - back][u, p]
        if top_r is not None:
            assert _topr_band(pstar[u], p, top_r), f"top-r decision differs at unit {u} page {p}"
            res.band_events += 1
            continue
        assert ps >= 0 and abs(ps - alpha) < BAND, (
            f"ts differs at unit {u} page {p}: gpu {g['ts'][u, p]} oracle {o['ts'][u, p]}, "
            f"p*={ps!r} outside the |p*-alpha|<{BAND} band")
        res.band_events += 1
    if resync:
        layer.raas_set_state(o["t"], o["ts"], o["start"], o["count"], o["pinned"])


def compare_sampled(layer, orc, units, alpha, pstar, res, top_r=None):
    """Full-size lockstep on sampled units: the oracle holds only `units` of the GPU handle.
    Their state must be bit-exact (a differing timestamp only inside the band, counted, then
    the GPU rows are resynced to the oracle's)."""
    gs = layer.raas_get_state()
    os_ = orc.get_state()
    g = {k: v[units] for k, v in gs.items()}
    same = all(np.array_equal(g[k], os_[k]) for k in os_)
    if same:
        return
    for k in ("t", "start", "count", "pinned"):
        assert np.array_equal(g[k], os_[k]), f"state field {k} differs outside the stamp band"
    for u, p in np.argwhere(g["ts"] != os_["ts"]):
        ps = pstar[u, p]
        if top_r is not None:
            assert _topr_band(pstar[u], p, top_r), f"top-r decision differs at sampled unit {units[u]} page {p}"
            res.band_events += 1
            continue
        assert ps >= 0 and abs(ps - alpha) < BAND, (
            f"ts differs at sampled unit {units[u]} page {p}: gpu {g['ts'][u, p]} oracle "
            f"{os_['ts'][u, p]}, p*={ps!r} outside the |p*-alpha|<{BAND} band")
        res.band_events += 1
    full = {k: v.copy() for k, v in gs.items()}
    full["ts"][units] = os_["ts"]
    layer.raas_set_state(full["t"], full["ts"], full["start"], full["count"], full["pinned"])


def run_lockstep(oracle_mod, stream, L, alpha, Hq, Hkv, split_pages=0, check_every=1,
                 layer=None, oracle=None, device="cuda", on_step=None, score_mode=0,
                 stamp_rule=0, top_r=0.5, quest_prefill_pages=0, table_scope=0, page=16,
                 state_every=1):
    """Drive both sides through the whole stream; returns LockstepResult.  Outputs are compared
    every `check_every` steps, the state every `state_every` of those (a state readout applies
    the token mode's deferred stamps, so sparse readouts exercise the deferred path)."""
    B, _, P, d = stream.k_pre.shape
    if layer is None:
        layer = RaasLayer(L, alpha, Hq, Hkv, d, B, device=device, split_pages=split_pages,
                          score_mode=score_mode, stamp_rule=stamp_rule, top_r=top_r,
                          quest_prefill_pages=quest_prefill_pages, table_scope=table_scope,
                          page=page)
        layer.raas_prefill(to_dev(stream.k_pre, device), to_dev(stream.v_pre, device), P)
    if oracle is None:
        oracle = oracle_mod.Oracle(L=L, alpha=alpha, page=page, n_q_heads=Hq, n_kv_heads=Hkv,
                                   head_dim=d, batch=B, score_mode=score_mode,
                                   stamp_rule=stamp_rule, top_r=top_r,
                                   quest_prefill_pages=quest_prefill_pages, table_scope=table_scope)
        oracle.prefill(stream.k_pre, stream.v_pre, P)
    res = LockstepResult()
    history = []
    out = torch.empty((B, Hq, d), dtype=torch.bfloat16, device=device)
    for i in range(stream.T):
        q, k, v = (to_dev(x[i], device) for x in (stream.q, stream.k, stream.v))
        layer.raas_decode_step(q, k, v, out)
        o_out = oracle.decode_step(stream.q[i], stream.k[i], stream.v[i])
        res.steps += 1
        if (i + 1) % check_every and i + 1 != stream.T:
            continue
        torch.cuda.synchronize()
        g_out = bf16_to_f32(from_dev(out)).astype(np.float64)
        assert np.isfinite(g_out).all()
        res.max_err = max(res.max_err, float(np.abs(g_out - o_out).max()))
        tr = oracle.get_trace()
        res.evictions += int((tr["evicted"] >= 0).sum())
        history.append(tr["pstar"].copy())
        if (i + 1) % (check_every * state_every) == 0 or i + 1 == stream.T:
            g_state = layer.raas_get_state()
            o_state = oracle.get_state()
            compare_state(g_state, o_state, alpha, tr["pstar"], res, layer,
                          top_r=top_r if stamp_rule == 1 else None,
                          history=history if state_every > 1 else None)
            history = []
        if on_step is not None:
            on_step(i, layer, oracle, g_out, o_out)
    assert layer.raas_get_status() == 0
    return res, layer, oracle
