#!/usr/bin/env python
"""bench.py — RaaS decode hot path on B200 (libraas), driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]
                    [--scaling weak|strong] [--shard requests|heads]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

`--gpus N` without torchrun (WORLD_SIZE unset) launches the N ranks itself (one process per
GPU, NCCL rendezvous on 127.0.0.1); under torchrun `--gpus` must equal WORLD_SIZE.

A "step" is one MODEL decode step: `layers` raas_decode_step launches (one per layer handle,
each a distinct 512 MiB KV cache at the headline config), i.e. every row of SURVEY.md §8(a)
for every request of this rank's batch.  Requests are sharded over ranks with no collective on
the hot path: `--scaling weak` (default) keeps the per-GPU batch fixed,
`--scaling strong` splits the config's global batch (config 4: 256 requests) over the ranks.
`--shard heads` splits the kv-heads instead (config 2, B = 1) with one NCCL all-gather of out
per layer-step, captured with the decode launches in one CUDA graph.

Rank 0 prints ONE JSON line.  `value` = model decode steps/s summed over GPUs (each step
decodes `per_gpu_batch` tokens per GPU); `e2e` = the same metric through
raas_decode_step_host (pinned host q/k/v in, out back to the host, copies inside the timed
region); `roofline` = algorithmic HBM bytes of one raas_decode_kernel launch / its average
duration vs MEASURED_PEAKS.json; `cpu_baseline` = the fp64 CPU oracle on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode steps/s and attention HBM GB/s (% of 8 TB/s) at L=2048, 1/2/4/8 B200"

# BASELINE.json configs (shapes from the public model configs)
CONFIGS = {
    1: dict(workload="toy_4q2kv_d64_L64", model="toy", hq=4, hkv=2, d=64, layers=1, batch=1,
            P=32, L=64, decode=256),
    2: dict(workload="llama31_8b_b1_L1024", model="Llama-3.1-8B attention (32q/8kv, d=128)",
            hq=32, hkv=8, d=128, layers=32, batch=1, P=512, L=1024, decode=8192, split_pages=16),
    3: dict(workload="llama31_8b_b64_L2048", model="Llama-3.1-8B attention (32q/8kv, d=128)",
            hq=32, hkv=8, d=128, layers=32, batch=64, P=256, L=2048, decode=16384),
    4: dict(workload="r1_distill_qwen7b_b32pergpu_L4096",
            model="DeepSeek-R1-Distill-Qwen-7B attention (28q/4kv, d=128)", hq=28, hkv=4, d=128,
            layers=28, batch=32, global_batch=256, P=128, L=4096, decode=32768),
    5: dict(workload="llama31_8b_b64_budget_sweep", model="Llama-3.1-8B attention (32q/8kv, d=128)",
            hq=32, hkv=8, d=128, layers=4, batch=64, P=128, L=2048, decode=32768),
}


UNIT = "decode steps/s"  # both arms (ours, --impl reference) print exactly this unit


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def unit_detail(B, nl, world, mode):
    """What one 'decode step' is in this run (the unit string itself is UNIT for every arm)."""
    if mode == "heads":
        return f"model steps of {B} request(s) x {nl} layers, kv-heads split over {world} GPUs"
    if mode == "strong":
        return f"model steps of the global batch ({B} requests over {world} GPUs) x {nl} layers"
    return f"model steps of {B} requests x {nl} layers per GPU, summed over {world} GPU(s)"


def free_port():
    import socket

    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    return port


def spawn_ranks(n, argv):
    """`--gpus N` without torchrun: start N ranks of this script (RANK / LOCAL_RANK /
    WORLD_SIZE / MASTER_* set as torchrun would, rendezvous on 127.0.0.1); rank 0's stdout is
    this process's.  A failing rank stops the others.  Returns the exit code."""
    import subprocess

    port = free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + argv, env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    while procs:
        for p_ in list(procs):
            code = p_.poll()
            if code is None:
                continue
            procs.remove(p_)
            if code != 0:
                rc = rc or code
                for q_ in procs:
                    q_.kill()
        time.sleep(0.05)
    return rc


# ----------------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, dev_index, period=0.02):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self._stop = period, threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            uuid_env = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = dev_index
            if uuid_env:
                vis = [x.strip() for x in uuid_env.split(",")]
                if dev_index < len(vis) and vis[dev_index].isdigit():
                    idx = int(vis[dev_index])
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            log("clock sampler unavailable:", e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------------- helpers
def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def variant_name(args):
    """The non-default method options of this run, '' for the default."""
    v = []
    if args.score != "exact":
        v.append(f"score={args.score}")
    if args.top_r > 0:
        v.append(f"top-r={args.top_r}")
    if args.table_scope:
        v.append("table=request")
    if args.page != 16:
        v.append(f"page={args.page}")
    if args.P:
        v.append(f"P={args.P}")
    if args.quest_prefill:
        v.append(f"hybrid K={args.quest_prefill}")
    if args.split_pages:
        v.append(f"split={args.split_pages}")
    return ", ".join(v)


def ncu_traffic(workload):
    """dram read+write bytes per launch of the dominant kernel, from the committed ncu
    summary (profiles/ncu_traffic.json, written from an `ncu --set full` capture)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


def cpu_count_info():
    try:
        n = len(os.sched_getaffinity(0))
    except Exception:
        n = os.cpu_count() or 1
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return n, model


def oracle_sample(cfg, seconds=12.0, max_steps=100000, seed=4242, threads=0):
    """Time the fp64 CPU oracle (as it stands) on a bounded sample of the workload: one layer,
    `threads` units of the config from a full-cache state, steady-state decode steps until
    `seconds` elapse.  threads = 0: every host core.  Returns unit-steps/s, the threads used and
    a description."""
    import numpy as np

    import oracle
    from paper_2502_11147_b200.synth import bf16_bits, random_steady_state

    ncores, cpu_model = cpu_count_info()
    threads = oracle.set_threads(threads if threads > 0 else ncores)
    g = cfg["hq"] // cfg["hkv"]
    C, Pp = cfg["L"] // 16, -(-cfg["P"] // 16)
    n_units = max(cfg["hkv"], (threads // cfg["hkv"]) * cfg["hkv"])
    nb = n_units // cfg["hkv"]
    d = cfg["d"]
    t_now = Pp * 16 + 4 * 16 * (C - Pp) + 1
    meta = random_steady_state(seed, n_units, C, Pp, t_now)
    rng = np.random.Generator(np.random.Philox(seed + 1))
    ks = bf16_bits(rng.standard_normal((n_units, C, 16, d), np.float32))
    vs = bf16_bits(rng.standard_normal((n_units, C, 16, d), np.float32))
    orc = oracle.Oracle(L=cfg["L"], alpha=1e-4, page=16, n_q_heads=nb * 0 + cfg["hq"],
                        n_kv_heads=cfg["hkv"], head_dim=d, batch=nb)
    orc.set_state(meta["t"], meta["ts"], meta["start"], meta["count"], meta["pinned"], ks, vs)
    steps = 0
    t0 = time.perf_counter()
    while steps < max_steps:
        q = bf16_bits(2.5 * rng.standard_normal((nb, cfg["hq"], d), np.float32))
        kn = bf16_bits(rng.standard_normal((nb, cfg["hkv"], d), np.float32))
        vn = bf16_bits(rng.standard_normal((nb, cfg["hkv"], d), np.float32))
        orc.decode_step(q, kn, vn)
        steps += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    orc.close()
    unit_steps_per_s = steps * n_units / dt
    desc = (f"{steps} steady-state decode steps of {n_units} units ({nb} requests x "
            f"{cfg['hkv']} kv-heads, g={g}, L={cfg['L']}, d={d}) of one layer from a full-cache "
            f"state, {dt:.1f} s on {threads} threads ({cpu_model}); extrapolated linearly to "
            f"{cfg['batch']} requests x {cfg['layers']} layers per step")
    return unit_steps_per_s, threads, desc


# ----------------------------------------------------------------------------------- main arm
def l2_rotation(cache_bytes_per_rot, l2_bytes, cap=64):
    """Distinct layer-cache sets cycled by consecutive steps so that the caches one step's
    timing can hit in L2 are >= 4x the L2 size (SURVEY §8(d) L2 hygiene); capped (toy)."""
    need = 4 * l2_bytes
    return max(1, min(cap, -(-need // max(1, cache_bytes_per_rot))))


def run_ours(args, cfg, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2502_11147_b200 import build as build_mod
    from paper_2502_11147_b200.raas import RaasLayer
    from paper_2502_11147_b200.shard import HeadGather, head_range, request_range

    if rank == 0 or not os.path.exists(build_mod.LIB):
        build_mod.build()
    if world > 1:
        torch.distributed.barrier()
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    hq, hkv, d, L, P, nl = cfg["hq"], cfg["hkv"], cfg["d"], cfg["L"], cfg["P"], cfg["layers"]
    heads = args.shard == "heads" and world > 1
    mode = "heads" if heads else args.scaling
    if heads and args.table_scope:
        raise SystemExit("--table-scope 1 shares one page table over a request's kv-heads; "
                         "shard by requests")
    B_global = cfg.get("global_batch", cfg["batch"]) if mode == "strong" else cfg["batch"] * world
    if mode == "strong":
        b_lo, b_hi = request_range(B_global, world, rank)
        B = b_hi - b_lo
        if B == 0:
            raise SystemExit(f"strong scaling: {B_global} requests leave rank {rank} idle")
    else:
        B = cfg["batch"]
    g = hq // hkv
    hq_full = hq
    if heads:  # this rank's kv-heads and their q-heads; out is all-gathered every layer-step
        kv_lo, kv_hi, q_lo, q_hi = head_range(hkv, hq, world, rank)
        hkv, hq = kv_hi - kv_lo, q_hi - q_lo
    C = L // 16
    Pp = -(-P // 16)
    units = B * hkv
    sp = args.split_pages if args.split_pages else cfg.get("split_pages", 0)
    score_mode = 1 if args.score == "quest" else 0
    # L2 hygiene: enough distinct layer-cache sets that consecutive steps never re-read L2
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    set_bytes = nl * 2 * units * C * 16 * d * 2
    rot = l2_rotation(set_bytes, l2) if args.rotate < 0 else max(1, args.rotate)
    layers = [RaasLayer(L, args.alpha, hq, hkv, d, B, device=dev, split_pages=sp, score_mode=score_mode,
                        stamp_rule=1 if args.top_r > 0 else 0, top_r=args.top_r,
                        quest_prefill_pages=args.quest_prefill, table_scope=args.table_scope,
                        page=args.page)
              for _ in range(nl * rot)]
    lay = lambda r: layers[r * nl:(r + 1) * nl]  # noqa: E731  (rotation r's layer handles)
    info = layers[0].raas_launch_info()
    # steady state before the timed region: fill the decode pages once, then a further page cycle
    fill_steps = (C - Pp) * 16 + 256 if args.fill < 0 else args.fill
    fill_steps = min(fill_steps, cfg["decode"])
    e_steps = max(4, min(args.steps, 64))
    # one distinct input slot (and graph) per warmup/timed step; slot s runs rotation s % rot
    R = -(-(args.warmup + args.steps) // rot) * rot
    if args.data == "gaussian":
        R = max(8, rot)  # i.i.d. inputs: a small ring suffices
    qs = [torch.empty((B, hq, d), device=dev, dtype=torch.bfloat16) for _ in range(R)]
    ks = [torch.empty((B, hkv, d), device=dev, dtype=torch.bfloat16) for _ in range(R)]
    vs = [torch.empty((B, hkv, d), device=dev, dtype=torch.bfloat16) for _ in range(R)]
    stream = torch.cuda.Stream(device=dev)
    seed = 1000 * args.config + rank
    if args.data == "waterfall":
        # PAPER.md §3.1 waterfall workload, drawn on the GPU step by step; each
        # rotation is its own stream (every layer of it sees the same draws: distinct caches)
        from paper_2502_11147_b200.synth import WaterfallTorch

        wfs = [WaterfallTorch(seed + 7919 * r, B, hq, hkv, d, P, fill_steps + R + e_steps + 8, dev,
                              lam=args.lam) for r in range(rot)]
        with torch.cuda.stream(stream):
            for r in range(rot):
                k, v = wfs[r].prefill()
                for ly in lay(r):
                    ly.raas_prefill(k, v, P, stream=stream)
        stream.synchronize()
        del k, v
        draw = lambda s_: wfs[s_ % rot].step(qs[s_], ks[s_], vs[s_])  # noqa: E731
    else:
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        for ly in layers:
            k = torch.randn((B, hkv, P, d), device=dev, generator=gen).bfloat16()
            v = torch.randn((B, hkv, P, d), device=dev, generator=gen).bfloat16()
            ly.raas_prefill(k, v, P)
            del k, v
        for s_ in range(R):
            qs[s_].copy_(torch.randn((B, hq, d), device=dev, generator=gen).mul_(2.5))
            ks[s_].copy_(torch.randn((B, hkv, d), device=dev, generator=gen))
            vs[s_].copy_(torch.randn((B, hkv, d), device=dev, generator=gen))
        draw = lambda s_: None  # noqa: E731
    outs = [torch.empty((B, hq, d), device=dev, dtype=torch.bfloat16) for _ in range(nl)]
    gathers = [HeadGather(B, hq, d, torch.bfloat16, dev) for _ in range(nl)] if heads else None

    def model_step(s_):  # one model step on input slot s_: nl launches (+ nl all-gathers)
        for li, ly in enumerate(lay(s_ % rot)):
            ly.raas_decode_step(qs[s_], ks[s_], vs[s_], outs[li], stream=stream)
            if heads:
                gathers[li](outs[li])

    # one CUDA graph per input slot, each = one model step (head sharding over NCCL: the
    # all-gathers are captured with the launches; gloo test mode runs eagerly)
    graphed = not heads or gathers[0].capturable
    graphs = []
    torch.cuda.synchronize()
    if graphed:
        with torch.cuda.stream(stream):
            for s in range(R):
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=stream):
                    model_step(s)
                graphs.append(gr)
    run_step = (lambda s_: graphs[s_].replay()) if graphed else model_step
    # capturing does not execute; fill now (real steps; every rotation advances fill_steps)
    t_fill = time.perf_counter()
    with torch.cuda.stream(stream):  # CUDAGraph.replay() launches on the current stream
        for i in range(fill_steps * rot):
            draw(i % R)
            run_step(i % R)
    torch.cuda.synchronize()
    t_fill = time.perf_counter() - t_fill
    c0 = [ly.raas_get_counters() for ly in layers]
    st0 = layers[0].raas_get_state()
    Ce = L // args.page  # state entries per unit: pages, or token slots (page = 1)
    log(f"[rank {rank}] filled {fill_steps} model steps x {rot} rotation(s) in {t_fill:.1f}s; used "
        f"entries/unit={(st0['count'] > 0).sum(1).mean():.1f}/{Ce}; batch {B}; launch {info}")

    # the warmup and timed steps' inputs, drawn before the timed region (slot i = step i)
    with torch.cuda.stream(stream):
        for i in range(R if args.data == "waterfall" else 0):
            draw(i)
    # warmup
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            run_step(i % R)
    torch.cuda.synchronize()
    if args.trace and rank == 0:
        # CUPTI kernel trace (torch.profiler / Kineto) of 2 model steps of the release build:
        # per-launch start / end inside the CUDA graphs, i.e. the PDL overlap (evidence only;
        # the number below is timed without the profiler)
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            with torch.cuda.stream(stream):
                for i in range(2):
                    run_step((args.warmup + i) % R)
            torch.cuda.synchronize()
        prof.export_chrome_trace(args.trace)
        log(f"[rank 0] kernel trace of 2 model steps -> {args.trace}")
    if world > 1:
        torch.distributed.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for i in range(args.steps):
                run_step((args.warmup + i) % R)
            ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    ms = ev0.elapsed_time(ev1)
    red_dev = dev if not world > 1 or torch.distributed.get_backend() == "nccl" else "cpu"
    per_rank = [ms]
    if world > 1:  # max over ranks (and every rank's own time, to show all ranks worked)
        t_all = torch.zeros(world, device=red_dev, dtype=torch.float64)
        t_all[rank] = ms
        torch.distributed.all_reduce(t_all)
        per_rank = [float(x) for x in t_all.cpu()]
    ms_max = max(per_rank)
    ms_per_step = ms_max / args.steps
    c1 = [ly.raas_get_counters() for ly in layers]
    stamps = sum(b_["stamps"] - a_["stamps"] for a_, b_ in zip(c0, c1))
    decisions = sum(b_["decisions"] - a_["decisions"] for a_, b_ in zip(c0, c1))
    evictions = sum(b_["evictions"] - a_["evictions"] for a_, b_ in zip(c0, c1))
    unit_steps = sum(b_["unit_steps"] - a_["unit_steps"] for a_, b_ in zip(c0, c1))
    status = max(ly.raas_get_status() for ly in layers)

    # algorithmic bytes per launch: K+V of resident tokens (steady state: the
    # write page holds 1..16 tokens, the others are full -> mean occupancy L-7.5 over a page
    # cycle; exact from the state at the timed steps), new K/V write, q read + out write,
    # metadata (ts/start/count) <= 12 B per entry (page, or token slot when page = 1).
    st1 = layers[0].raas_get_state()
    occ_now = st1["count"].sum(1).mean()
    if (st0["count"] > 0).sum(1).min() == Ce:
        occ_mean = L - 7.5 if args.page == 16 else float(L)  # token slots: always all L
    else:
        occ_mean = float(occ_now)
    nfull = P // 16
    # Quest score mode: every attended page also brings its min / max key rows (2 of 32 rows:
    # "+1/16 bytes read"), maintained on write
    qtr = 4 * d * (occ_mean / 16) if args.score == "quest" and args.page == 16 else 0.0
    if args.quest_prefill and nfull > args.quest_prefill:
        # hybrid: only K of the nfull prompt pages are read, plus their representative keys
        occ_mean -= (nfull - args.quest_prefill) * 16
        bytes_launch = units * (4 * d * occ_mean + 4 * d + 4 * g * d + 12 * Ce + nfull * 4 * d + qtr)
    else:
        bytes_launch = units * (4 * d * occ_mean + 4 * d + 4 * g * d + 12 * Ce + qtr)
    variant = bool(args.score != "exact" or args.top_r > 0 or args.table_scope or args.page != 16
                   or args.quest_prefill or args.P or args.L or args.batch or args.layers
                   or args.split_pages or args.dense or heads or mode == "strong")
    launch_s = ms_per_step / 1e3 / nl
    achieved = bytes_launch / launch_s / 1e9
    peak, peak_src = measured_peaks()
    if achieved > 1.3 * peak:
        raise RuntimeError(f"achieved {achieved:.0f} GB/s > 1.3x the copy peak: the timed region "
                           "did not do the work")
    model_steps_per_s = args.steps / (ms_max / 1e3)
    # weak: every GPU steps its own batch -> summed; strong / heads: one global step per period
    value = model_steps_per_s * (world if mode == "weak" else 1)
    tokens_per_s = model_steps_per_s * (B * world if mode == "weak" else B_global if mode == "strong" else B)

    # ---------------- e2e: through raas_decode_step_host with pinned host buffers -------
    e2e = None
    if not args.no_e2e and not heads:
        # each e2e step has its own inputs (the stream continues), staged in pinned host memory;
        # every layer's call copies them H2D and its out D2H inside the timed region
        ne = e_steps + 2
        hq_ = torch.empty((ne, B, hq, d), dtype=torch.bfloat16).pin_memory()
        hk_ = torch.empty((ne, B, hkv, d), dtype=torch.bfloat16).pin_memory()
        hv_ = torch.empty((ne, B, hkv, d), dtype=torch.bfloat16).pin_memory()
        ho_ = [torch.empty((B, hq, d), dtype=torch.bfloat16).pin_memory() for _ in range(nl)]
        with torch.cuda.stream(stream):
            for j in range(ne):
                draw(j % R)
                hq_[j].copy_(qs[j % R])
                hk_[j].copy_(ks[j % R])
                hv_[j].copy_(vs[j % R])
        stream.synchronize()
        e_next = [0]

        def e2e_step():  # one stream: H2D, step, D2H of every layer in order (no overlap)
            j = e_next[0]
            e_next[0] += 1
            for li, ly in enumerate(lay(j % rot)):
                ly.raas_decode_step_host(hq_[j], hk_[j], hv_[j], ho_[li], stream=stream)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(e_steps):
            e2e_step()
        e1.record(stream)
        stream.synchronize()
        wall = time.perf_counter() - w0
        e_ms = max(e0.elapsed_time(e1), wall * 1e3)
        te = torch.tensor([e_ms], device=red_dev, dtype=torch.float64)
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": e_steps / (float(te.item()) / 1e3) * (world if mode == "weak" else 1),
               "unit": UNIT, "steps": e_steps,
               "h2d_bytes_per_step": nl * (B * hq * d + 2 * B * hkv * d) * 2 * world,
               "d2h_bytes_per_step": nl * B * hq * d * 2 * world,
               "api": "raas_decode_step_host (pinned host q/k_new/v_new -> out: zero-copy ingest kernel + out stored to host by the combine), one stream, layers in order"}

    if rank != 0:
        return None
    cache_bytes = rot * set_bytes  # this rank's K/V stores over all layer handles
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        ups, threads, desc = oracle_sample(cfg, seconds=args.cpu_seconds)
        ups1, _, desc1 = oracle_sample(cfg, seconds=max(2.0, args.cpu_seconds / 4), threads=1)
        cpu = {"value": ups / (units * nl), "unit": UNIT, "cores": threads,
               "kind": "oracle", "sample": desc, "unit_steps_per_s": ups,
               "single_thread": {"value": ups1 / (units * nl), "unit": UNIT, "cores": 1,
                                 "unit_steps_per_s": ups1, "sample": desc1}}
    l2_note = (f"{nl * rot} distinct layer caches ({rot} rotation(s) of {nl}) = "
               f"{cache_bytes / 2**30:.3f} GiB vs L2 {l2 / 2**20:.0f} MiB: "
               + (f">= 4x L2, consecutive steps read disjoint caches (no flush needed)"
                  if cache_bytes >= 4 * l2 else "< 4x L2: part of the K/V stream can hit in L2"))
    out = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak" if mode == "weak" else "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": (f"synthetic waterfall stream (PAPER.md §3.1 / DESIGN.md §4: sink + 2 recent pages, "
                 f"milestones, phoenix; page-correlated keys; lambda={args.lam}), seeded torch Philox "
                 "on the GPU, bf16, a distinct input per step" if args.data == "waterfall" else
                 "synthetic (seeded torch Philox; K/V ~ N(0,1), q ~ N(0, 2.5^2), bf16)"),
        "config": {"workload": cfg["workload"], "model_shapes": cfg["model"], "layers": nl,
                   "unit_detail": unit_detail(B_global if mode == "strong" else B, nl, world, mode),
                   "per_gpu_batch": B, "global_batch": B_global if not heads else B,
                   "prefill": P, "L": L,
                   "page": args.page, "alpha": args.alpha, "score_mode": args.score,
                   "stamp_rule": f"top-r {args.top_r}" if args.top_r > 0 else "alpha",
                   "quest_prefill_pages": args.quest_prefill,
                   "table_scope": "request" if args.table_scope else "kv-head",
                   "variant": variant_name(args),
                   "parallelism": (f"head-sharded x{world}: kv-heads split, NCCL all-gather of out per "
                                   f"layer-step{' (in the CUDA graph)' if graphed else ' (eager, gloo)'}"
                                   if heads else
                                   f"request-sharded x{world} ({mode} scaling), no collective"),
                   "l2": l2_note,
                   "steady_state": f"{fill_steps} decode steps before warmup (all pages used, evicting)"},
        "tokens_per_s": tokens_per_s,
        "achieved_note": ("per-GPU HBM figures; the roofline covers this rank's decode launches"
                          if world > 1 else None),
        "per_rank_ms": per_rank,
        "layer_steps_per_s": value * nl,
        "hbm_gbs": achieved,
        "pct_of_8tbs": achieved / 8000.0 * 100.0,
        "pct_of_measured_copy": achieved / peak * 100.0,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     # the committed ncu capture is of the default variant of the workload
                     "traffic": None if variant else ncu_traffic(cfg["workload"]),
                     "kernel": f"raas_decode_kernel<{d},8,16> grid {info['grid']} x {info['block']} thr, "
                               f"{info['smem']} B smem, {info['split_pages']}-page splits"
                               + (f", clusters of {info['cluster']} (partials via DSMEM)" if info['cluster'] > 1 else ""),
                     "algorithmic_bytes_per_launch": bytes_launch,
                     "avg_launch_us": launch_s * 1e6, "peak_source": peak_src,
                     "timing": "CUDA events on the launch stream around K graph replays of "
                               f"{nl} launches; avg launch = step / {nl}"},
        "e2e": e2e,
        "gpu_launches": args.steps * nl * (2 if args.quest_prefill else 1) * world,
        "launch": info,
        "stamp_rate": stamps / max(decisions, 1),
        "evictions_per_step": evictions / max(unit_steps, 1) * units,
        "device_status": status,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    return out


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle (as it stands) on a bounded sample, same metric, unit and
    config as our arm.  Under N ranks, rank 0 alone works and prints; the others join the
    process group (gloo, CPU), wait at the barriers and exit 0."""
    import torch

    if world > 1:
        torch.distributed.init_process_group("gloo")
        torch.distributed.barrier()
    out = None
    if rank == 0:
        units = cfg["batch"] * cfg["hkv"]
        t0 = time.perf_counter()
        ups, threads, desc = oracle_sample(cfg, seconds=args.cpu_seconds)
        wall = time.perf_counter() - t0
        v = ups / (units * cfg["layers"])
        out = {
            "impl": "reference",
            "metric": METRIC,
            "value": v,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (full-cache state, seeded Philox, bf16 values; the oracle's bounded sample)",
            "config": {"workload": cfg["workload"], "model_shapes": cfg["model"],
                       "unit_detail": unit_detail(cfg["batch"], cfg["layers"], 1, "weak"),
                       "per_gpu_batch": cfg["batch"], "L": cfg["L"], "prefill": cfg["P"],
                       "layers": cfg["layers"],
                       "parallelism": "rank 0 only (the oracle on the host cores)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall,
        }
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--alpha", type=float, default=1e-4)
    ap.add_argument("--L", type=int, default=0, help="override the budget (config 5 sweep)")
    ap.add_argument("--batch", type=int, default=0, help="override the per-GPU (weak) / global (strong) batch")
    ap.add_argument("--layers", type=int, default=0, help="override the layer count")
    ap.add_argument("--fill", type=int, default=-1, help="decode steps before warmup (-1: auto)")
    ap.add_argument("--data", default="waterfall", choices=["waterfall", "gaussian"],
                    help="input stream: the waterfall workload (default) or i.i.d. Gaussian")
    ap.add_argument("--lam", type=float, default=7.0,
                    help="waterfall query strength (7: ~50%% page stamp rate at config 3)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="requests", choices=["requests", "heads"],
                    help="multi-GPU: shard requests (no collective) or kv-heads (all-gather of out)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="request sharding: fixed per-GPU batch (weak) or fixed global batch (strong)")
    ap.add_argument("--rotate", type=int, default=-1,
                    help="layer-cache rotations (-1: enough for >= 4x L2 of distinct caches)")
    ap.add_argument("--split-pages", type=int, default=0, help="override pages per split tile")
    ap.add_argument("--quest-prefill", type=int, default=0,
                    help="Quest-on-prefill hybrid: prompt pages attended per step (NEXT-4)")
    ap.add_argument("--P", type=int, default=0, help="override the prompt length")
    ap.add_argument("--top-r", type=float, default=0.0,
                    help="stamp the top r fraction of pages instead of the alpha threshold (NEXT-3)")
    ap.add_argument("--score", default="exact", choices=["exact", "quest"],
                    help="page score for stamping: exact page max (D4) or Quest bound (NEXT-1)")
    ap.add_argument("--page", type=int, default=16, choices=[16, 1],
                    help="1: token-level RaaS (PAPER.md §3.2), one timestamp per token (NEXT-3)")
    ap.add_argument("--table-scope", type=int, default=0, choices=[0, 1],
                    help="1: one page table per request, OR over all heads (reading D25)")
    ap.add_argument("--trace", default="",
                    help="write a CUPTI kernel trace (chrome json) of 2 model steps before timing")
    ap.add_argument("--dense", type=int, default=0,
                    help="dense comparator: prefill N tokens, L > N + steps (no eviction)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus, sys.argv[1:]))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    cfg = dict(CONFIGS[args.config])
    if args.L:
        cfg["L"] = args.L
        cfg["workload"] += f"_L{args.L}"
    if args.dense:  # dense decode comparator (P1): the whole context resident, nothing evicted
        cfg["P"] = args.dense
        cfg["L"] = ((args.dense + args.warmup + args.steps + 64) // 16 + 1) * 16
        cfg["workload"] += f"_dense_N{args.dense}"
        args.fill = 0
    if args.batch:
        cfg["batch"] = args.batch
        cfg["global_batch"] = args.batch
    if args.P:
        cfg["P"] = args.P
        cfg["workload"] += f"_P{args.P}"
    if args.layers:
        cfg["layers"] = args.layers
    if args.scaling == "strong" and args.shard == "requests":
        cfg["workload"] = cfg["workload"].replace("_b32pergpu", "") + f"_strong_b{cfg.get('global_batch', cfg['batch'])}"
    args.warmup = max(args.warmup, 3)

    # RAAS_BENCH_SHARE_GPU=1: test mode for the multi-rank path on a single GPU (ranks share
    # device 0, gloo carries the barriers and the timing reduction); never a bench number
    share = os.environ.get("RAAS_BENCH_SHARE_GPU") == "1"
    if args.impl == "reference":
        out = run_reference(args, cfg, rank, world)
    else:
        import torch

        if share:
            local_rank = local_rank % torch.cuda.device_count()
        if world > 1:
            torch.cuda.set_device(local_rank)
            if share:
                torch.distributed.init_process_group("gloo")
            else:
                torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        out = run_ours(args, cfg, rank, world, local_rank)
        if share and out is not None:
            out["note"] = "RAAS_BENCH_SHARE_GPU test mode: ranks shared one GPU; not a measurement"
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
