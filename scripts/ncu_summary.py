#!/usr/bin/env python
"""Summarise an ncu report of raas_decode_kernel: headline counters + warp-stall samples by
source line (needs the .so the report was taken with, for SASS -> line mapping).

    python scripts/ncu_summary.py gpurun_out/prof_v2.ncu-rep [--lib paper_2502_11147_b200/libraas.so]
"""
import argparse
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__inst_executed_pipe_tensor.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    # SURVEY §8(d)'s list: tensor pipe (confirms the MMAs), long-scoreboard share, achieved
    # occupancy (= sm__warps_active.avg.pct_of_peak_sustained_active)
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "sm__maximum_warps_per_active_cycle_pct",
]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw_metrics(rep):
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for i, h in enumerate(hdr):
        if h in METRICS or h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            out[h] = (vals[i], units[i])
    return out


def stall_by_line(rep, lib, kernel_regex):
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "source", "--csv",
                                            "--print-source", "sass"]))))
    hdr = rows[1]
    ia, iss = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    prof = [(int(r[ia], 16), int(r[iss] or 0)) for r in rows[2:] if len(r) > iss and r[ia].startswith("0x")]
    base = prof[0][0]
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=td, capture_output=True)
        cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
        sass = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(td, cub)],
                              capture_output=True, text=True).stdout.split("\n")
    start = [i for i, l in enumerate(sass) if re.match(r"\.text\.\S*" + kernel_regex, l)][0]
    cur, off2 = None, {}
    for l in sass[start + 1:]:
        if l.startswith(".text."):
            break
        m = re.search(r'## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        m2 = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m2:
            off2[int(m2.group(1), 16)] = cur
    agg = {}
    for a, n in prof:
        k = off2.get(a - base)
        agg[k] = agg.get(k, 0) + n
    return agg


def mangled_from_report(rep):
    """Mangled name of the profiled raas_decode_kernel instantiation, from the report's demangled
    'raas_decode_kernel<128, 8, 16, 0, 0, 0, 0>' (D, NC, S, TOKD, GEN, CL[, FM])."""
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    name = rows[2][rows[0].index("Kernel Name")]
    args = [int(x) for x in re.search(r"<([^>]*)>", name).group(1).split(",")]
    kinds = ["i", "i", "i", "b", "b", "b", "i"][:len(args)]
    body = "".join(f"L{k}{v}E" for k, v in zip(kinds, args))
    return f"_ZN4raas18raas_decode_kernelI{body}EEvNS_12DecodeParamsE"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--lib", default="paper_2502_11147_b200/libraas.so")
    ap.add_argument("--kernel", default="",
                    help="mangled-name regex of the profiled instantiation (default: from the report)")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    m = raw_metrics(a.rep)
    print("## counters")
    for k in METRICS:
        if k in m:
            print(f"- {k}: {m[k][0]} {m[k][1]}")
    st = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: int(float(v[0])) for k, v in m.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_")}
    tot = sum(st.values()) or 1
    print("\n## stall reasons (pc samples)")
    for k, v in sorted(st.items(), key=lambda x: -x[1])[:12]:
        print(f"- {k}: {v} ({100 * v / tot:.1f}%)")
    kern = a.kernel or mangled_from_report(a.rep)
    print(f"\n(source lines mapped through {kern} in {a.lib})")
    try:
        agg = stall_by_line(a.rep, a.lib, re.escape(kern) if not a.kernel else kern)
    except Exception as e:  # pragma: no cover
        print("(no line mapping:", e, ")")
        return
    root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2502_11147_b200", "csrc")
    files = {}
    tot = sum(agg.values()) or 1
    print("\n## stall samples by source line")
    for k, n in sorted(agg.items(), key=lambda x: -x[1])[:a.top]:
        txt = "?"
        if k:
            fn = os.path.join(root, k[0])
            if os.path.exists(fn):
                files.setdefault(fn, open(fn).read().split("\n"))
                txt = files[fn][k[1] - 1].strip()[:90]
        print(f"- {n:5d} {100 * n / tot:5.1f}%  {k[0] if k else '?'}:{k[1] if k else ''}  `{txt}`")


if __name__ == "__main__":
    sys.exit(main())
