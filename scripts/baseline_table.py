"""Markdown table of measured bench lines (BASELINE.md §2 'Measured'): the headline JSON plus
the configs JSON lines.   python scripts/baseline_table.py profiles/r01_bench_cfg3.json profiles/r01_configs.jsonl"""
import json
import sys


def lines(path):
    with open(path) as f:
        for ln in f:
            ln = ln.strip()
            if ln.startswith("{"):
                yield json.loads(ln)


DEFAULT_P = {"llama31_8b_b64_L2048": 256}


def variant(c):
    if "variant" in c:
        return c["variant"] or "—"
    v = []  # lines written before bench.py recorded the variant
    if c.get("score_mode", "exact") != "exact":
        v.append(f"score={c['score_mode']}")
    if str(c.get("stamp_rule", "alpha")) != "alpha":
        v.append(str(c["stamp_rule"]).replace(" ", "="))
    if c.get("table_scope", "kv-head") != "kv-head":
        v.append("table=request")
    if c.get("page", 16) != 16:
        v.append(f"page={c['page']}")
    if c["workload"] in DEFAULT_P and c.get("prefill") != DEFAULT_P[c["workload"]]:
        v.append(f"P={c['prefill']}")
    if c.get("quest_prefill_pages"):
        v.append(f"hybrid K={c['quest_prefill_pages']}")
    return ", ".join(v) or "—"


# the GPU parity test (tests/test_gpu_parity.py) that runs each workload's shapes in the launch
# configuration bench.py times
PARITY = {
    "llama31_8b_b64_L2048": "full-size lockstep (cfg 3 x2) + bench-stream lockstep",
    "llama31_8b_b1_L1024": "full-size lockstep (cfg 2) + cluster-vs-default bitwise",
    "r1_distill_qwen7b_b32pergpu_L4096": "full-size lockstep (cfg 4)",
    "llama31_8b_b64_budget_sweep_L8192": "full-size lockstep (cfg 5, L = 8192)",
    "llama31_8b_b64_budget_sweep_L256": "full-size lockstep (cfg 5, L = 256)",
}


def parity(c):
    v = variant(c)
    if v == "—":
        return PARITY.get(c["workload"], "small-config lockstep (same kernel, other shapes)")
    return "variant lockstep (small configs)"


rows = []
for p in sys.argv[1:]:
    rows.extend(lines(p))
print("| workload | variant | B/GPU | L | layers | µs/layer-step | model-steps/s | tokens/s "
      "| GB/s (algorithmic) | % of measured peak | % of 8 TB/s | stamp rate | evictions / layer-step "
      "| e2e model-steps/s | SM MHz | parity |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for d in rows:
    c, r = d["config"], d["roofline"]
    us = d["ms_per_step"] * 1e3 / c["layers"]
    e2e = d.get("e2e") or {}
    print(f"| {c['workload']} | {variant(c)} | {c['per_gpu_batch']} | {c['L']} | {c['layers']} "
          f"| {us:.1f} | {d['value']:.1f} | {d.get('tokens_per_s', 0):.0f} "
          f"| {r['achieved']:.0f} | {100 * r['frac']:.1f} | {100 * r['achieved'] / 8000:.1f} "
          f"| {100 * d.get('stamp_rate', 0):.0f} % | {d.get('evictions_per_step', 0):.1f} "
          f"| {e2e.get('value', float('nan')):.1f} | {d.get('clocks', {}).get('sm_mhz', '')} | {parity(c)} |")
