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


rows = []
for p in sys.argv[1:]:
    rows.extend(lines(p))
print("| workload | variant | B/GPU | L | layers | ms/step | µs/layer-step | model-steps/s | tokens/s "
      "| GB/s (algorithmic) | % of measured peak | % of 8 TB/s | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for d in rows:
    c, r = d["config"], d["roofline"]
    us = d["ms_per_step"] * 1e3 / c["layers"]
    print(f"| {c['workload']} | {variant(c)} | {c['per_gpu_batch']} | {c['L']} | {c['layers']} "
          f"| {d['ms_per_step']:.3f} | {us:.1f} | {d['value']:.1f} | {d.get('tokens_per_s', 0):.0f} "
          f"| {r['achieved']:.0f} | {100 * r['frac']:.1f} | {100 * r['achieved'] / 8000:.1f} "
          f"| {d.get('clocks', {}).get('sm_mhz', '')} |")
