"""Markdown table of bench.py JSON lines: rows/s and roofline fraction per mode.
usage: python scripts/summarize_bench.py file.json [file.json ...]"""
import json
import sys


def main(paths):
    print("| file | workload | rows/GPU | SHAP rows/s | SHAP frac | interactions rows/s | interactions frac | "
          "e2e rows/s | CPU oracle rows/s (cores) | SM MHz |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        try:
            d = json.loads(open(p).read().strip().splitlines()[-1])
        except Exception:
            continue
        if "config" not in d:
            continue
        c = d["config"]
        s, i = d.get("shap") or {}, d.get("interactions") or {}
        cpu = d.get("cpu_baseline") or {}
        e2e = d.get("e2e") or {}
        f = lambda x: f"{x:.4g}" if isinstance(x, (int, float)) and x else "–"
        fr = lambda m: f"{(m.get('roofline') or {}).get('frac', 0):.3f}" if m else "–"
        print(f"| {p.split('/')[-1]} | {c.get('workload')} | {c.get('rows_per_gpu')} | {f(s.get('rows_per_s'))} | "
              f"{fr(s)} | {f(i.get('rows_per_s'))} | {fr(i)} | {f(e2e.get('value'))} | "
              f"{f(cpu.get('value'))} ({cpu.get('cores', '–')}) | {(d.get('clocks') or {}).get('sm_mhz')} |")


if __name__ == "__main__":
    main(sys.argv[1:])
