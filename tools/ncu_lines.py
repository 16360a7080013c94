"""Per-source-line instruction and stall breakdown of one kernel from an ncu
report (`ncu --page source --print-source cuda,sass`): the lines that issue
the most warp instructions, with their share and top stall samples.

    python tools/ncu_lines.py REPORT KERNEL_REGEX [launch_skip] [top]
"""
import csv
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                          f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur_file = ""
    agg = []
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or (len(r) > 2 and r[2] != "-"):
            continue   # source-line rows only (SASS rows carry an address)
        try:
            ie = float(r[hdr.index("Instructions Executed")].replace(",", "") or 0)
            ss = float(r[hdr.index("Warp Stall Sampling (All Samples)")].replace(",", "") or 0)
        except (ValueError, IndexError):
            continue
        if ie > 0:
            agg.append((ie, ss, f"{cur_file}:{r[0]}", r[1].strip()[:90]))
    tot = sum(a[0] for a in agg) or 1
    tss = sum(a[1] for a in agg) or 1
    print(f"total warp instructions {tot:.4g}, stall samples {tss:.4g}")
    for ie, ss, loc, src in sorted(agg, reverse=True)[:top]:
        print(f"{100 * ie / tot:6.2f}% inst {100 * ss / tss:6.2f}% samples  {loc:22s} {src}")


if __name__ == "__main__":
    main()
