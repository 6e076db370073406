#!/usr/bin/env python
"""Summarise a bench.py --trace kernel trace (CUPTI via torch.profiler, release build): every
decode launch's start / end on the device, the overlap of consecutive launches (programmatic
dependent launch lets launch k+1 start before launch k ends), and the launch period, to set
beside ncu's serialised per-launch time and bench.py's CUDA-event step time.

    python scripts/trace_summary.py gpurun_out/trace_cfg3.json [--layers 32]
"""
import argparse
import json
import statistics


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("trace")
    ap.add_argument("--layers", type=int, default=32)
    a = ap.parse_args()
    ev = json.load(open(a.trace))
    ev = ev["traceEvents"] if isinstance(ev, dict) else ev
    ks = sorted((e for e in ev if e.get("cat") == "kernel" and "raas_decode_kernel" in e.get("name", "")),
                key=lambda e: e["ts"])
    other = sorted((e for e in ev if e.get("cat") == "kernel" and "raas_decode_kernel" not in e.get("name", "")),
                   key=lambda e: e["ts"])
    if not ks:
        raise SystemExit("no raas_decode_kernel events")
    t0 = ks[0]["ts"]
    dur = [e["dur"] for e in ks]
    starts = [e["ts"] for e in ks]
    ends = [e["ts"] + e["dur"] for e in ks]
    ov = [ends[i] - starts[i + 1] for i in range(len(ks) - 1)]
    period = (ends[-1] - starts[0]) / len(ks)
    print(f"decode launches: {len(ks)} (other kernels in the window: {len(other)})")
    print(f"per-launch device duration (start -> end, overlapping neighbours): median {statistics.median(dur):.1f} us, "
          f"min {min(dur):.1f}, max {max(dur):.1f}")
    print(f"overlap of launch k's end with launch k+1's start: median {statistics.median(ov):.1f} us "
          f"(positive = k+1 started before k ended)")
    print(f"period (first start -> last end) / launches: {period:.1f} us")
    if other:
        od = [e["dur"] for e in other]
        names = sorted({e["name"].split("(")[0][:60] for e in other})
        print(f"other kernels: {len(other)}, median {statistics.median(od):.1f} us ({', '.join(names)})")
    print("first launches (us from the first start): start, end, duration")
    for e in ks[: min(len(ks), 6)]:
        print(f"  {e['ts'] - t0:9.1f} {e['ts'] + e['dur'] - t0:9.1f} {e['dur']:7.1f}")


if __name__ == "__main__":
    main()
