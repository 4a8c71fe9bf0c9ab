"""Instruction mix (executed warp instructions by opcode) per kernel from an
ncu report's source page.  Usage: python scripts/ncu_sass_mix.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            secs.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and len(r) > 5:
            cur["rows"].append(r)
    seen = set()
    for s in secs:
        if s["name"] in seen:
            continue
        seen.add(s["name"])
        I = {h: i for i, h in enumerate(s["hdr"])}
        data = [r for r in s["rows"] if r[I["Instructions Executed"]].isdigit()]
        tot = sum(int(r[I["Instructions Executed"]]) for r in data)
        ops, stall = collections.Counter(), collections.Counter()
        for r in data:
            t = r[I["Source"]].split()
            if not t:
                continue
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            ops[op] += int(r[I["Instructions Executed"]])
            stall[op] += int(r[I["Warp Stall Sampling (All Samples)"]] or 0)
        print(f"{s['name'][:90]}  executed warp instrs {tot:.3e}")
        for k, v in ops.most_common(int(top)):
            print(f"   {k:10s} {v:14d} {v / max(tot, 1) * 100:5.1f}%   stall samples {stall[k]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
