"""Copy one GPU session's evidence from gpurun_out/<tag>/ into profiles/<name>/:
the bench line, the ncu launch list with per-kernel shares, the ncu --set full
summaries, test logs; and record per-launch DRAM traffic in profiles/traffic.json
(read by bench.py for roofline.traffic).

usage: python scripts/collect_profiles.py gpurun_out/r01a profiles/r01 [workload/layout/mode/dtype=kernelregex[@capture][#rows] ...]
"""
import collections
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys


def launch_shares(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        agg.setdefault(r[ki], []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values()) or 1.0
    out = ["kernel | launches | total ms | mean ms/launch | share of device time",
           "---|---|---|---|---"]
    for k, v in agg.items():
        out.append(f"{k} | {len(v)} | {sum(v) / 1e6:.3f} | {sum(v) / len(v) / 1e6:.4f} | {sum(v) / tot:.4f}")
    return "\n".join(out) + "\n"


def rep_traffic(rep):
    """{kernel name: [dram read+write bytes per launch, ...]} from an ncu report."""
    if rep.endswith(".raw.csv"):
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return {}
    hdr, units = rows[0], rows[1]
    res = collections.defaultdict(list)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for r in rows[2:]:
        try:
            b = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(m)
                b += float(r[i].replace(",", "")) * scale.get(units[i], 1)
            res[r[hdr.index("Kernel Name")]].append(b)
        except (ValueError, IndexError):
            continue
    return res


def main():
    src, dst = sys.argv[1], sys.argv[2]
    keys = [a.split("=", 1) for a in sys.argv[3:] if "=" in a]
    os.makedirs(dst, exist_ok=True)
    for f in sorted(os.listdir(src)):
        p = os.path.join(src, f)
        if f.endswith(".ncu-rep") or f.endswith(".raw.csv") or os.path.isdir(p):
            continue
        if f.endswith(".csv") and "launch" in f:
            open(os.path.join(dst, f.replace(".csv", ".shares.md")), "w").write(launch_shares(p))
        shutil.copy(p, os.path.join(dst, f))
    tfile = os.path.join(os.path.dirname(dst.rstrip("/")), "traffic.json")
    traffic = json.load(open(tfile)) if os.path.exists(tfile) else {}
    reps = [f for f in os.listdir(src) if f.endswith(".ncu-rep")]
    reps += [f for f in os.listdir(src) if f.endswith(".raw.csv") and f[:-8] + ".ncu-rep" not in reps]
    for rep in sorted(reps):
        tr = rep_traffic(os.path.join(src, rep))
        rep = rep[:-8] + ".ncu-rep" if rep.endswith(".raw.csv") else rep
        for key, rx in keys:
            rx, _, rows = rx.partition("#")  # key=kernelregex[@capture][#rows]: rows per captured launch
            rx, _, only = rx.partition("@")  # key=kernelregex@capture: only that capture's kernels
            if only and not rep.startswith(only):
                continue
            for kname, vals in tr.items():
                if re.search(rx, kname) and vals and all(v == v for v in vals):
                    traffic[key] = {"dram_bytes_per_launch": sum(vals) / len(vals), "kernel": kname,
                                    "source": f"{dst}/{rep[:-8]}.summary.txt (ncu --set full, dram__bytes_read.sum + "
                                              f"dram__bytes_write.sum)", "launches": len(vals)}
                    if rows:
                        traffic[key]["rows_per_launch"] = int(rows)
    json.dump(traffic, open(tfile, "w"), indent=1, sort_keys=True)
    print(open(tfile).read())


if __name__ == "__main__":
    main()
