#!/bin/bash
# Bench every BASELINE workload on one GPU (SHAP + interactions where in scope).
set -u
OUT=gpurun_out/${TAG:-all}
mkdir -p $OUT
run() { local name=$1; shift; timeout 1200 python bench.py --workload "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$?"; }
run cal_housing-small cal_housing-small --rows-per-gpu 1048576 --steps 10 --no-ablation ${EXTRA:-}
run cal_housing-med cal_housing-med --rows-per-gpu 1048576 --steps 10 ${EXTRA:-}
run cal_housing-med-f64 cal_housing-med --rows-per-gpu 262144 --steps 5 --dtype f64 --no-ablation ${EXTRA:-}
run adult-large adult-large --rows-per-gpu 65536 --steps 5 ${EXTRA:-}
run fashion_mnist-med fashion_mnist-med --rows-per-gpu 65536 --steps 5 --mode shap --x-layout feature ${EXTRA:-}
run fashion_mnist-med-rowmajor fashion_mnist-med --rows-per-gpu 65536 --steps 5 --mode shap --no-ablation ${EXTRA:-}
run fashion_mnist-med-int fashion_mnist-med --rows-per-gpu 10000 --steps 3 --mode interactions --no-ablation ${EXTRA:-}
run covtype-large covtype-large --rows-per-gpu 32768 --steps 3 --mode shap ${EXTRA:-}
run covtype-large-int covtype-large --rows-per-gpu 8192 --steps 3 --mode interactions --no-ablation ${EXTRA:-}
run depth3-single depth3-single --rows-per-gpu 100 --steps 20 --no-ablation --no-e2e ${EXTRA:-}
python - <<'PY'
import json, glob, os
for f in sorted(glob.glob(os.environ.get("OUT", "gpurun_out/all") + "/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    s = d.get("shap") or {}; i = d.get("interactions") or {}
    print(f"{os.path.basename(f):28s} value {d['value']:.4g} rows/s | shap {s.get('rows_per_s', 0):.4g} frac {((s.get('roofline') or {}).get('frac') or 0):.3f} | "
          f"inter {i.get('rows_per_s', 0):.4g} frac {((i.get('roofline') or {}).get('frac') or 0):.3f} | cpu {((d.get('cpu_baseline') or {}).get('value') or 0):.4g} | e2e {((d.get('e2e') or {}).get('value') or 0):.4g}")
PY
