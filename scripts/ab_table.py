"""Summarise gpu_ab.sh JSON lines: lib x workload -> rows/s (frac) per mode."""
import glob
import json
import os
import sys

for d in sys.argv[1:]:
    for f in sorted(glob.glob(os.path.join(d, "*.json"))):
        try:
            j = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception as e:  # noqa: BLE001
            print(os.path.basename(f), "ERR", e)
            continue
        parts = []
        for m in ("shap", "interactions", "both"):
            x = j.get(m)
            if isinstance(x, dict) and "rows_per_s" in x:
                parts.append(f"{m} {x['rows_per_s']:.4g} ({x['roofline']['frac']:.3f})")
        if not parts:
            parts.append(f"value {j.get('value', 0):.4g} ({j.get('roofline', {}).get('frac', 0):.3f})")
        print(f"{os.path.basename(f):55s} " + "  ".join(parts))
