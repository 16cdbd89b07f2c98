"""Warp-stall breakdown per kernel of an `ncu --set full` report: the top
smsp__average_warps_issue_stalled_<reason>_per_issue_active.ratio values (warps stalled per
issue-active cycle), with the kernel's time, issue-active and warps-active percentages.

usage: python scripts/ncu_stalls.py gpurun_out/prof_full.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head = rows[0]
    name_i = head.index("Kernel Name")
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    stall_cols = [(i, h[len(pre):-len(suf)]) for i, h in enumerate(head) if h.startswith(pre) and h.endswith(suf)]
    col = {h: i for i, h in enumerate(head)}
    seen = set()
    for r in rows[2:]:
        name = r[name_i]
        if name in seen:
            continue
        seen.add(name)
        t = num(r[col["gpu__time_duration.sum"]])
        ia = num(r[col["smsp__issue_active.avg.pct_of_peak_sustained_active"]])
        wa = num(r[col["sm__warps_active.avg.pct_of_peak_sustained_active"]])
        inst = num(r[col["smsp__inst_executed.sum"]])
        st = sorted(((num(r[i]) or 0.0, n) for i, n in stall_cols), reverse=True)[:top]
        print(f"== {name[:70]}  {t:.3f} ms, issue-active {ia:.1f}%, warps active {wa:.1f}%, {inst / 1e9:.3f} G warp-inst")
        print("   " + ", ".join(f"{n} {v:.2f}" for v, n in st))


if __name__ == "__main__":
    main()
