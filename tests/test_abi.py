"""CPU checks of the C ABI boundary: libraas.so builds for sm_100a, loads without a GPU,
exports every function include/raas.h declares, and rejects bad arguments before touching
the device."""
import ctypes
import os
import shutil

import pytest

from paper_2502_11147_b200 import build as build_mod
from paper_2502_11147_b200 import raas

HAVE_NVCC = shutil.which("nvcc") is not None or os.path.exists("/usr/local/cuda/bin/nvcc")


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(raas.LIB_PATH):
        if not HAVE_NVCC:
            pytest.skip("no nvcc and no prebuilt libraas.so")
        build_mod.build()
    return raas.lib()


def test_header_symbols_exported(L):
    names = raas.header_functions()
    assert "raas_create" in names and "raas_decode_step" in names and "raas_prefill" in names
    assert "raas_destroy" in names
    for n in names:
        assert hasattr(L, n), f"{n} declared in include/raas.h but not exported"
    # nothing else named raas_* is exported
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", raas.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = sorted({ln.split()[-1] for ln in out.splitlines() if " T raas_" in ln})
    assert exported == names


def test_sass_is_sm100a_and_uses_bulk_copies_and_tensor_cores(L):
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump) and not shutil.which("cuobjdump"):
        pytest.skip("no cuobjdump")
    import subprocess

    sass = subprocess.run([cuobjdump, "-sass", raas.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    assert "UBLKCP" in sass             # bulk async copies (TMA engine) of the KV pages
    assert "HMMA.16816.F32.BF16" in sass  # bf16 tensor-core MMAs (QK^T and PV)
    assert "LDSM" in sass and "MOVM" in sass


def test_sass_cluster_instantiation_uses_cluster_barriers(L):
    """The small-batch cluster schedule's kernel (raas_decode_kernel<..., CL = true>) carries the
    thread-block-cluster barrier (barrier.cluster -> UCGABAR) and remote mbarrier arrivals on the
    leader (mbarrier.arrive.release.cluster -> SYNCS.ARRIVE...RED); the default lean kernel
    carries none of it."""
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump) and not shutil.which("cuobjdump"):
        pytest.skip("no cuobjdump")
    import subprocess

    def sass(fn):
        return subprocess.run([cuobjdump, "-sass", "-fun", fn, raas.LIB_PATH], capture_output=True,
                              text=True).stdout
    cl = sass("_ZN4raas18raas_decode_kernelILi128ELi8ELi16ELb0ELb0ELb1ELi0EEEvNS_12DecodeParamsE")
    lean = sass("_ZN4raas18raas_decode_kernelILi128ELi8ELi16ELb0ELb0ELb0ELi0EEEvNS_12DecodeParamsE")
    assert "UCGABAR_ARV" in cl and "UCGABAR_WAIT" in cl and "SYNCS.ARRIVE.TRANS64.RED" in cl
    assert "HMMA.16816.F32.BF16" in cl and "UBLKCP" in cl
    assert lean and "UCGABAR" not in lean


@pytest.mark.parametrize("cfg,expect", [
    (dict(L=64, alpha=1e-4, n_q_heads=4, n_kv_heads=2, head_dim=64, batch=1), True),
    (dict(L=2048, alpha=1e-4, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=64), True),
    (dict(L=50, alpha=1e-4, n_q_heads=4, n_kv_heads=2, head_dim=64, batch=1), False),   # L % 16
    (dict(L=64, alpha=1e-4, n_q_heads=5, n_kv_heads=2, head_dim=64, batch=1), False),   # Hq % Hkv
    (dict(L=64, alpha=1e-4, n_q_heads=4, n_kv_heads=2, head_dim=96, batch=1), False),   # head_dim
    (dict(L=64, alpha=1e-4, n_q_heads=32, n_kv_heads=2, head_dim=64, batch=1), False),  # group 16
    (dict(L=64, alpha=-1.0, n_q_heads=4, n_kv_heads=2, head_dim=64, batch=1), False),   # alpha < 0
])
def test_arena_bytes(L, cfg, expect):
    n = raas.raas_arena_bytes(raas.make_config(**cfg))
    assert (n > 0) == expect
    if expect:
        C, U = cfg["L"] // 16, cfg["batch"] * cfg["n_kv_heads"]
        kv = 2 * U * C * 16 * cfg["head_dim"] * 2
        assert kv <= n <= kv * 1.2 + (1 << 20)   # O(L): the KV store dominates


@pytest.mark.parametrize("extra", [dict(score_mode=2), dict(stamp_rule=3), dict(stamp_rule=1, top_r=1.5),
                                   dict(quest_prefill_pages=-1), dict(split_pages=33),
                                   dict(stamp_rule=1, top_r=0.5, L=16384),
                                   dict(quest_prefill_pages=8, L=16384), dict(table_scope=2),
                                   dict(page=8), dict(page=1, L=2040), dict(page=1, score_mode=1),
                                   dict(page=1, quest_prefill_pages=4),
                                   dict(page=1, stamp_rule=1, L=1024), dict(disable_early_start=2),
                                   dict(L=80 * 32 * 16 + 16)])   # > MAX_SPLITS x 32-page splits
def test_arena_bytes_rejects_bad_modes(L, extra):
    base = dict(L=2048, alpha=1e-4, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=2)
    base.update(extra)
    assert raas.raas_arena_bytes(raas.make_config(**base)) == 0


def test_hybrid_mode_adds_representative_keys_only(L):
    base = dict(L=2048, alpha=1e-4, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=2)
    a0 = raas.raas_arena_bytes(raas.make_config(**base))
    a1 = raas.raas_arena_bytes(raas.make_config(**base, quest_prefill_pages=16))
    kv = 2 * 16 * 128 * 2 * 2 * 128 * 16   # units x pages x (K+V rows) bytes
    assert 0 < a1 - a0 <= kv / 16 + 2 * 16 * 128 * 4 + 4096   # min/max keys (1/16 of K) + vmap


def test_token_level_arena(L):
    """page = 1: the same KV store (plus a 128-byte ts/start trailer per 16-row tile in the
    deferred mode), metadata per token instead of per page."""
    base = dict(L=2048, alpha=1e-4, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=2)
    a16 = raas.raas_arena_bytes(raas.make_config(**base))
    a1 = raas.raas_arena_bytes(raas.make_config(**base, page=1))
    units, tiles, extra_entries = 16, 128, 2048 - 128
    meta = units * extra_entries * 3 * 4                   # ts / start / cnt per token
    assert meta <= a1 - a16 <= meta + units * tiles * 128 + 1024 * 1024
    # the non-deferred token path (top-r) keeps every token's score per head
    a1r = raas.raas_arena_bytes(raas.make_config(**dict(base, L=512, page=1, stamp_rule=1)))
    a16r = raas.raas_arena_bytes(raas.make_config(**dict(base, L=512, stamp_rule=1)))
    assert a1r - a16r >= units * (512 - 32) * (3 * 4 + 4 * 4)


def test_arena_is_linear_in_L_not_N(L):
    """Memory plateaus at the budget (PAPER.md :191-193): the arena depends on L only."""
    a = [raas.raas_arena_bytes(raas.make_config(L=L_, alpha=1e-4, n_q_heads=32, n_kv_heads=8,
                                                head_dim=128, batch=4)) for L_ in (512, 1024, 2048)]
    assert a[1] - a[0] == pytest.approx(a[2] - a[1], rel=0.02) or a[2] - a[1] == pytest.approx(2 * (a[1] - a[0]), rel=0.05)


def test_create_rejects_bad_args_without_gpu(L):
    cfg = raas.make_config(L=64, alpha=1e-4, n_q_heads=4, n_kv_heads=2, head_dim=64, batch=1)
    h = ctypes.c_void_p()
    n = raas.raas_arena_bytes(cfg)
    assert L.raas_create(ctypes.byref(cfg), ctypes.c_void_p(1024), n - 1, 0, ctypes.byref(h)) == raas.RAAS_E_ARENA
    assert L.raas_create(ctypes.byref(cfg), ctypes.c_void_p(1025), n, 0, ctypes.byref(h)) == raas.RAAS_E_ARENA
    assert L.raas_create(ctypes.byref(cfg), None, n, 0, ctypes.byref(h)) == raas.RAAS_E_ARENA
    bad = raas.make_config(L=64, alpha=1e-4, n_q_heads=4, n_kv_heads=2, head_dim=80, batch=1)
    assert L.raas_create(ctypes.byref(bad), ctypes.c_void_p(1024), 1 << 30, 0, ctypes.byref(h)) == raas.RAAS_E_UNSUPPORTED
    assert b"head_dim" in L.raas_last_error()
    assert L.raas_decode_step(None, None, None, None, None, None) == raas.RAAS_E_INVALID
    assert L.raas_prefill(None, None, None, 0, None) == raas.RAAS_E_INVALID


def test_quest_mode_adds_min_max_rows_per_page(L):
    """score_mode 1 keeps every page's per-channel min / max key rows (Quest's representative
    keys, PAPER.md :147) in the page's HBM trailer: 2 rows per 32 K/V rows (+6.25 % bytes)."""
    base = dict(L=2048, alpha=1e-4, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=2)
    a0 = raas.raas_arena_bytes(raas.make_config(**base))
    a1 = raas.raas_arena_bytes(raas.make_config(**base, score_mode=1))
    units, pages = 16, 128
    trailer = units * pages * 2 * 128 * 2
    assert trailer <= a1 - a0 <= trailer + 4096
