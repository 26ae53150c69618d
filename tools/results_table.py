"""Markdown results table from a bench JSONL file (default profiles/r01_bench_all_configs.jsonl)."""
import json
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_bench_all_configs.jsonl"
print("| config | mode | impl | evals/s | ms/pass | scaling | e2e evals/s | CPU oracle evals/s (1 core) "
      "| dominant kernel: achieved / peak (frac) |")
print("|---|---|---|---|---|---|---|---|---|")
for ln in open(path):
    d = json.loads(ln)
    c = d["config"]
    r = d.get("roofline") or {}
    dom = "-"
    if r.get("kernel"):
        if r.get("achieved") is not None:
            dom = f"{r['kernel']}: {r['achieved']:.3g} / {r['peak']:.4g} {r['unit']} ({r['frac']:.3f})"
        else:
            dom = f"{r['kernel']}: latency-bound"
    cpu = (d.get("cpu_baseline") or {}).get("value")
    print(f"| {c['workload'][:2]} | {c['mode']} | {d.get('impl', 'ours')} | {d['value']:.4g} | {d['ms_per_step']:.4f} "
          f"| {d['scaling']} | {d['e2e']['value']:.4g} | {cpu:.4g} | {dom} |" if cpu else
          f"| {c['workload'][:2]} | {c['mode']} | {d.get('impl', 'ours')} | {d['value']:.4g} | {d['ms_per_step']:.4f} "
          f"| {d['scaling']} | {d['e2e']['value']:.4g} | - | {dom} |")
