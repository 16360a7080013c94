"""SASS opcode mix of one kernel from an ncu report (executed warp
instructions per opcode and their share), e.g.

    python tools/ncu_sass_mix.py REPORT kk_pairs [launch_skip]
"""
import csv
import subprocess
import sys
from collections import defaultdict


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                          f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Address")
    si, ii, wi = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    agg = defaultdict(lambda: [0.0, 0.0])
    for r in rows:
        if len(r) != len(hdr) or r[0] in ("Address", "") or r[si] in ("...",):
            continue
        try:
            n = float(r[ii].replace(",", ""))
            w = float(r[wi].replace(",", ""))
        except ValueError:
            continue
        op = r[si].split()[0] if r[si].split() else "?"
        if op.startswith("@"):
            op = r[si].split()[1]
        agg[op.split(".")[0]][0] += n
        agg[op.split(".")[0]][1] += w
    tot = sum(v[0] for v in agg.values()) or 1
    tw = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {tot:.5g}")
    for op, (n, w) in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
        print(f"{op:10s} {100 * n / tot:6.2f}% inst  {100 * w / tw:6.2f}% stall samples")


if __name__ == "__main__":
    main()
