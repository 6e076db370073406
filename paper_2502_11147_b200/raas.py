"""Thin Python binding of libraas (include/raas.h) — argument marshalling only.

Every step of the decode path runs in libraas.so's CUDA kernels; PyTorch only provides
device memory (the arena, q/k/v/out tensors) and streams.  There is no fallback: if the
shared library is missing, ``lib()`` raises.

The C functions are exposed under their C names (``raas_create``, ``raas_prefill``,
``raas_decode_step``, ...); ``RaasLayer`` bundles one handle with its arena.
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RAAS_LIB may point at an alternative build of the same library (tuning experiments only)
LIB_PATH = os.environ.get("RAAS_LIB") or os.path.join(_HERE, "libraas.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "raas.h")

RAAS_OK, RAAS_E_INVALID, RAAS_E_UNSUPPORTED, RAAS_E_STATE, RAAS_E_BUDGET, RAAS_E_CUDA, RAAS_E_ARENA = range(7)


class raas_config(ctypes.Structure):
    _fields_ = [
        ("L", ctypes.c_int32),
        ("alpha", ctypes.c_float),
        ("page", ctypes.c_int32),
        ("n_q_heads", ctypes.c_int32),
        ("n_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("batch", ctypes.c_int32),
        ("softmax_scale", ctypes.c_float),
        ("split_pages", ctypes.c_int32),
        ("score_mode", ctypes.c_int32),
        ("stamp_rule", ctypes.c_int32),
        ("top_r", ctypes.c_float),
        ("quest_prefill_pages", ctypes.c_int32),
        ("table_scope", ctypes.c_int32),
        ("disable_early_start", ctypes.c_int32),
    ]


class RaasError(RuntimeError):
    def __init__(self, code: int, what: str):
        msg = lib().raas_last_error().decode(errors="replace")
        super().__init__(f"{what} -> {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libraas.so (built by ``paper_2502_11147_b200.build`` / ``__graft_entry__.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libraas.so not found at {LIB_PATH}: run `python -m paper_2502_11147_b200.build` "
            "(there is no CPU fallback)")
    l = ctypes.CDLL(LIB_PATH)
    V, I, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    l.raas_arena_bytes.argtypes = [ctypes.POINTER(raas_config)]
    l.raas_arena_bytes.restype = SZ
    l.raas_create.argtypes = [ctypes.POINTER(raas_config), V, SZ, I, ctypes.POINTER(V)]
    l.raas_prefill.argtypes = [V, V, V, ctypes.c_int32, V]
    l.raas_prefill_varlen.argtypes = [V, V, V, V, ctypes.c_int32, V]
    l.raas_decode_step.argtypes = [V, V, V, V, V, V]
    l.raas_decode_step_host.argtypes = [V, V, V, V, V, V]
    l.raas_destroy.argtypes = [V]
    l.raas_get_state.argtypes = [V, V, V, V, V, V, V]
    l.raas_set_state.argtypes = [V, V, V, V, V, V, V, V, V]
    l.raas_get_kv.argtypes = [V, V, V, V]
    l.raas_get_status.argtypes = [V, V]
    l.raas_get_counters.argtypes = [V, V, V]
    l.raas_launch_info.argtypes = [V, V]
    l.raas_last_error.argtypes = []
    l.raas_last_error.restype = ctypes.c_char_p
    for n in ("raas_create", "raas_prefill", "raas_prefill_varlen", "raas_decode_step", "raas_decode_step_host",
              "raas_destroy", "raas_get_state", "raas_set_state", "raas_get_kv",
              "raas_get_status", "raas_get_counters", "raas_launch_info"):
        getattr(l, n).restype = I
    _lib = l
    return l


def header_functions(path: str = HEADER):
    """Names of the functions include/raas.h declares."""
    src = open(path).read()
    return sorted(set(re.findall(r"RAAS_API\s+[\w\s\*]+?\b(raas_\w+)\s*\(", src)))


def _check(rc, what):
    if rc != RAAS_OK:
        raise RaasError(rc, what)


SCORE_EXACT, SCORE_QUEST = 0, 1
STAMP_ALPHA, STAMP_TOP_R = 0, 1


def make_config(L, alpha, n_q_heads, n_kv_heads, head_dim, batch, page=16, softmax_scale=0.0,
                split_pages=0, score_mode=SCORE_EXACT, stamp_rule=STAMP_ALPHA,
                top_r=0.5, quest_prefill_pages=0, table_scope=0,
                disable_early_start=0) -> raas_config:
    return raas_config(L, alpha, page, n_q_heads, n_kv_heads, head_dim, batch, softmax_scale,
                       split_pages, score_mode, stamp_rule, top_r, quest_prefill_pages, table_scope,
                       disable_early_start)


def raas_arena_bytes(cfg: raas_config) -> int:
    return int(lib().raas_arena_bytes(ctypes.byref(cfg)))


def _dptr(t):
    """Device pointer of a torch tensor (must be contiguous)."""
    if t is None:
        return None
    assert t.is_contiguous(), "tensor must be contiguous"
    return ctypes.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    if stream is None:
        import torch

        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _np_ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class RaasLayer:
    """One libraas handle (one attention layer of `batch` requests) plus its device arena."""

    def __init__(self, L, alpha, n_q_heads, n_kv_heads, head_dim, batch, device=None,
                 softmax_scale=0.0, split_pages=0, score_mode=SCORE_EXACT,
                 stamp_rule=STAMP_ALPHA, top_r=0.5, quest_prefill_pages=0, table_scope=0,
                 page=16, disable_early_start=0):
        import torch

        self.cfg = make_config(L, alpha, n_q_heads, n_kv_heads, head_dim, batch, page=page,
                               softmax_scale=softmax_scale, split_pages=split_pages,
                               score_mode=score_mode, stamp_rule=stamp_rule, top_r=top_r,
                               quest_prefill_pages=quest_prefill_pages, table_scope=table_scope,
                               disable_early_start=disable_early_start)
        self.device = torch.device(device if device is not None else "cuda")
        dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        nbytes = raas_arena_bytes(self.cfg)
        if nbytes == 0:
            raise RaasError(RAAS_E_INVALID, "raas_arena_bytes")
        # over-allocate for 1024-byte alignment
        self._arena_t = torch.empty(nbytes + 1024, dtype=torch.uint8, device=self.device)
        base = self._arena_t.data_ptr()
        off = (-base) % 1024
        self.arena_ptr = base + off
        self.arena_bytes = nbytes
        h = ctypes.c_void_p()
        _check(lib().raas_create(ctypes.byref(self.cfg), ctypes.c_void_p(self.arena_ptr),
                                 nbytes, dev_index, ctypes.byref(h)), "raas_create")
        self._h = h
        # state arrays have one entry per page (page = 16) or per token slot (page = 1)
        self.L, self.page, self.C = L, page, L // page
        self.hq, self.hkv, self.d, self.batch = n_q_heads, n_kv_heads, head_dim, batch
        self.units = batch * n_kv_heads

    # ---- the path -------------------------------------------------------------------
    def raas_prefill(self, k, v, P=None, stream=None):
        P = k.shape[2] if P is None else P
        _check(lib().raas_prefill(self._h, _dptr(k), _dptr(v), int(P), _stream_ptr(stream)),
               "raas_prefill")

    def raas_prefill_varlen(self, k, v, P_per_request, stream=None):
        """k, v: [batch, n_kv_heads, P_max, head_dim]; request b uses its first P[b] tokens."""
        P = np.ascontiguousarray(P_per_request, dtype=np.int32)
        assert P.shape == (self.batch,)
        _check(lib().raas_prefill_varlen(self._h, _dptr(k), _dptr(v), _np_ptr(P), int(k.shape[2]),
                                         _stream_ptr(stream)), "raas_prefill_varlen")

    def raas_decode_step(self, q, k_new, v_new, out, stream=None):
        _check(lib().raas_decode_step(self._h, _dptr(q), _dptr(k_new), _dptr(v_new), _dptr(out),
                                      _stream_ptr(stream)), "raas_decode_step")

    def raas_decode_step_host(self, q_host, k_host, v_host, out_host, stream=None):
        """Host (ideally pinned) torch tensors; copies are inside the call, async on stream."""
        for t in (q_host, k_host, v_host, out_host):
            assert t.device.type == "cpu" and t.is_contiguous()
        _check(lib().raas_decode_step_host(
            self._h, ctypes.c_void_p(q_host.data_ptr()), ctypes.c_void_p(k_host.data_ptr()),
            ctypes.c_void_p(v_host.data_ptr()), ctypes.c_void_p(out_host.data_ptr()),
            _stream_ptr(stream)), "raas_decode_step_host")

    # ---- introspection ----------------------------------------------------------------
    def raas_get_state(self, stream=None):
        U, C = self.units, self.C
        t = np.zeros(U, np.int32)
        ts = np.zeros((U, C), np.int32)
        st = np.zeros((U, C), np.int32)
        cnt = np.zeros((U, C), np.int32)
        pin = np.zeros((U, C), np.uint8)
        _check(lib().raas_get_state(self._h, _np_ptr(t), _np_ptr(ts), _np_ptr(st), _np_ptr(cnt),
                                    _np_ptr(pin), _stream_ptr(stream)), "raas_get_state")
        return dict(t=t, ts=ts, start=st, count=cnt, pinned=pin)

    def raas_set_state(self, t, ts, start, count, pinned, k_store=None, v_store=None, stream=None):
        a = [np.ascontiguousarray(x, dtype=np.int32) for x in (t, ts, start, count)]
        pin = np.ascontiguousarray(pinned, dtype=np.uint8)
        ks = None if k_store is None else np.ascontiguousarray(k_store, dtype=np.uint16)
        vs = None if v_store is None else np.ascontiguousarray(v_store, dtype=np.uint16)
        _check(lib().raas_set_state(self._h, *[_np_ptr(x) for x in a], _np_ptr(pin), _np_ptr(ks),
                                    _np_ptr(vs), _stream_ptr(stream)), "raas_set_state")

    def raas_get_kv(self, stream=None):
        shape = (self.units, self.C, self.page, self.d)
        k = np.zeros(shape, np.uint16)
        v = np.zeros(shape, np.uint16)
        _check(lib().raas_get_kv(self._h, _np_ptr(k), _np_ptr(v), _stream_ptr(stream)), "raas_get_kv")
        return k, v

    def raas_get_status(self, stream=None):
        rc = lib().raas_get_status(self._h, _stream_ptr(stream))
        if rc < 0:
            raise RaasError(-rc, "raas_get_status")
        return rc

    def raas_get_counters(self, stream=None):
        c = np.zeros(4, np.uint64)
        _check(lib().raas_get_counters(self._h, _np_ptr(c), _stream_ptr(stream)), "raas_get_counters")
        return dict(stamps=int(c[0]), decisions=int(c[1]), evictions=int(c[2]), unit_steps=int(c[3]))

    def raas_launch_info(self):
        i = np.zeros(6, np.int32)
        _check(lib().raas_launch_info(self._h, _np_ptr(i)), "raas_launch_info")
        return dict(grid=int(i[0]), block=int(i[1]), smem=int(i[2]), split_pages=int(i[3]),
                    nsplit=int(i[4]), cluster=int(i[5]))

    def close(self):
        if getattr(self, "_h", None):
            lib().raas_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
