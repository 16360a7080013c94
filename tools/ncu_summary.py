"""Summarise ncu outputs for profiles/: launch-list shares and full-set key
metrics (duration, DRAM bytes, issue/warps active, top stalls)."""
import csv
import subprocess
import sys
from collections import defaultdict


def launch_shares(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    names = [(r[ki], float(r[vi].replace(",", ""))) for r in data if len(r) > vi]
    starts = [i for i, (n, _) in enumerate(names) if "kk_pairs_kernel" in n]
    # one device-resident step: from the longest K1 launch (the whole 2^30
    # sample super-frame) to the next K1 launch
    s0 = max(starts, key=lambda i: names[i][1])
    nxt = [i for i in starts if i > s0]
    seg = names[s0:nxt[0]] if nxt else names[s0:]
    agg = defaultdict(lambda: [0, 0.0])
    for n, v in seg:
        agg[n.split("(")[0][:60]][0] += 1
        agg[n.split("(")[0][:60]][1] += v
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# one bench step, ncu gpu__time_duration (serialised, cold cache); total {tot/1e6:.3f} ms\n")
        f.write("share_pct,launches,ms,kernel\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{v[1]/tot*100:.2f},{v[0]},{v[1]/1e6:.4f},{k}\n")


def full_summary(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
    with open(out, "w") as f:
        for r in rows[2:]:
            f.write(f"== {r[h.index('Kernel Name')]}\n")
            for k in keys:
                if k in h:
                    f.write(f"   {k} = {r[h.index(k)]} {units[h.index(k)]}\n")
            st = []
            for i, c in enumerate(h):
                if c.startswith("smsp__pcsamp_warps_issue_stalled") and not c.endswith("not_issued"):
                    try:
                        st.append((float(r[i].replace(",", "")), c.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                    except ValueError:
                        pass
            tot = sum(v for v, _ in st) or 1
            f.write("   stalls: " + ", ".join(f"{c}={v/tot*100:.0f}%" for v, c in sorted(st, reverse=True)[:7]) + "\n")


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    (launch_shares if kind == "launches" else full_summary)(src, dst)
