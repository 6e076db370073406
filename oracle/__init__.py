"""CPU oracle for the RaaS decode hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product path
(``paper_2502_11147_b200``, ``libraas.so``) never imports it and shares no code with it.

This module is a thin ctypes loader for ``raas_ref.c`` (plain C, fp64), which follows
PAPER.md §3.3 / App. B step by step (see the C file for citations and DESIGN.md §3 for
the readings D1-D24).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "raas_ref.c")
_LIB = os.path.join(_HERE, "liboracle_raas.so")

REF_OK, REF_E_INVALID, REF_E_STATE, REF_E_BUDGET = 0, 1, 3, 4


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (OpenMP over units)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "raas_ref.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-Wall",
             "-Wno-unknown-pragmas", _SRC, "-o", tmp, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


class _Cfg(ctypes.Structure):
    _fields_ = [
        ("L", ctypes.c_int32),
        ("alpha", ctypes.c_double),
        ("page", ctypes.c_int32),
        ("n_q_heads", ctypes.c_int32),
        ("n_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("batch", ctypes.c_int32),
        ("softmax_scale", ctypes.c_double),
        ("score_mode", ctypes.c_int32),
        ("stamp_rule", ctypes.c_int32),
        ("top_r", ctypes.c_double),
        ("quest_prefill_pages", ctypes.c_int32),
        ("table_scope", ctypes.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        l = ctypes.CDLL(build())
        P = ctypes.c_void_p
        l.raas_ref_create.argtypes = [ctypes.POINTER(_Cfg), ctypes.POINTER(P)]
        l.raas_ref_destroy.argtypes = [P]
        l.raas_ref_destroy.restype = None
        l.raas_ref_prefill.argtypes = [P, P, P, ctypes.c_int32]
        l.raas_ref_prefill_varlen.argtypes = [P, P, P, P, ctypes.c_int32]
        l.raas_ref_decode_step.argtypes = [P, P, P, P, P]
        l.raas_ref_step_stamps.argtypes = [P, P]
        l.raas_ref_get_state.argtypes = [P, P, P, P, P, P]
        l.raas_ref_set_state.argtypes = [P, P, P, P, P, P, P, P]
        l.raas_ref_get_trace.argtypes = [P, P, P, P]
        l.raas_ref_get_kv.argtypes = [P, P, P]
        l.raas_ref_resident_positions.argtypes = [P, ctypes.c_int32, P, ctypes.c_int32]
        l.raas_ref_get_selection.argtypes = [P, P, P]
        l.raas_ref_set_threads.argtypes = [ctypes.c_int]
        _lib = l
    return _lib


def set_threads(n: int) -> int:
    return lib().raas_ref_set_threads(n)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what} failed with code {code}")
        self.code = code


class Oracle:
    """fp64 RaaS state machine over `batch * n_kv_heads` independent units (host)."""

    def __init__(self, L, alpha, page, n_q_heads, n_kv_heads, head_dim, batch,
                 softmax_scale=0.0, score_mode=0, stamp_rule=0, top_r=0.5,
                 quest_prefill_pages=0, table_scope=0):
        self.cfg = _Cfg(L, alpha, page, n_q_heads, n_kv_heads, head_dim, batch, softmax_scale,
                        score_mode, stamp_rule, top_r, quest_prefill_pages, table_scope)
        self.C = L // page if page > 0 else 0
        self.units = batch * n_kv_heads
        self.page, self.d, self.hq, self.hkv, self.batch = page, head_dim, n_q_heads, n_kv_heads, batch
        h = ctypes.c_void_p()
        rc = lib().raas_ref_create(ctypes.byref(self.cfg), ctypes.byref(h))
        if rc:
            raise OracleError(rc, "raas_ref_create")
        self._h = h

    def close(self):
        if self._h:
            lib().raas_ref_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _u16(a):
        a = np.ascontiguousarray(a)
        assert a.dtype == np.uint16, a.dtype
        return a

    def prefill(self, k_bits, v_bits, P):
        k = self._u16(k_bits) if P else None
        v = self._u16(v_bits) if P else None
        rc = lib().raas_ref_prefill(self._h, _ptr(k), _ptr(v), int(P))
        if rc:
            raise OracleError(rc, "raas_ref_prefill")

    def prefill_varlen(self, k_bits, v_bits, P_per_request):
        P = np.ascontiguousarray(P_per_request, dtype=np.int32)
        k, v = self._u16(k_bits), self._u16(v_bits)
        rc = lib().raas_ref_prefill_varlen(self._h, _ptr(k), _ptr(v), _ptr(P), int(k.shape[2]))
        if rc:
            raise OracleError(rc, "raas_ref_prefill_varlen")

    def decode_step(self, q_bits, k_bits, v_bits, want_out=True):
        q, k, v = self._u16(q_bits), self._u16(k_bits), self._u16(v_bits)
        out = np.zeros((self.batch, self.hq, self.d), np.float64) if want_out else None
        rc = lib().raas_ref_decode_step(self._h, _ptr(q), _ptr(k), _ptr(v), _ptr(out))
        if rc:
            raise OracleError(rc, "raas_ref_decode_step")
        return out

    def step_stamps(self, stamps):
        s = np.ascontiguousarray(stamps, dtype=np.uint8).reshape(self.units, self.C)
        rc = lib().raas_ref_step_stamps(self._h, _ptr(s))
        if rc:
            raise OracleError(rc, "raas_ref_step_stamps")

    def get_state(self):
        U, C = self.units, self.C
        t = np.zeros(U, np.int32)
        ts = np.zeros((U, C), np.int32)
        st = np.zeros((U, C), np.int32)
        cnt = np.zeros((U, C), np.int32)
        pin = np.zeros((U, C), np.uint8)
        lib().raas_ref_get_state(self._h, _ptr(t), _ptr(ts), _ptr(st), _ptr(cnt), _ptr(pin))
        return dict(t=t, ts=ts, start=st, count=cnt, pinned=pin)

    def set_state(self, t, ts, start, count, pinned, k_store=None, v_store=None):
        a = [np.ascontiguousarray(x, dtype=np.int32) for x in (t, ts, start, count)]
        pin = np.ascontiguousarray(pinned, dtype=np.uint8)
        ks = None if k_store is None else self._u16(k_store)
        vs = None if v_store is None else self._u16(v_store)
        rc = lib().raas_ref_set_state(self._h, *[_ptr(x) for x in a], _ptr(pin), _ptr(ks), _ptr(vs))
        if rc:
            raise OracleError(rc, "raas_ref_set_state")

    def get_kv(self):
        """K and V stores as bf16 bits [units][C][page][head_dim]."""
        shape = (self.units, self.C, self.page, self.d)
        ks, vs = np.zeros(shape, np.uint16), np.zeros(shape, np.uint16)
        rc = lib().raas_ref_get_kv(self._h, _ptr(ks), _ptr(vs))
        if rc:
            raise OracleError(rc, "raas_ref_get_kv")
        return ks, vs

    def get_trace(self):
        U, C = self.units, self.C
        ev = np.zeros(U, np.int32)
        sl = np.zeros(U, np.int32)
        ps = np.zeros((U, C), np.float64)
        lib().raas_ref_get_trace(self._h, _ptr(ev), _ptr(sl), _ptr(ps))
        return dict(evicted=ev, slot=sl, pstar=ps)

    def get_selection(self):
        U, C = self.units, self.C
        att = np.zeros((U, C), np.uint8)
        qs = np.zeros((U, C), np.float64)
        lib().raas_ref_get_selection(self._h, _ptr(att), _ptr(qs))
        return dict(attended=att, qscore=qs)

    def resident_positions(self, unit):
        cap = self.C * self.page
        pos = np.zeros(cap, np.int32)
        n = lib().raas_ref_resident_positions(self._h, int(unit), _ptr(pos), cap)
        return pos[:n].copy()
