"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel name, launches,
summed time and share of the total (cold-cache, serialized launch times: compare shares).

usage: python scripts/launch_shares.py gpurun_out/launches.csv [header note]
"""
import csv
import io
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    note = sys.argv[2] if len(sys.argv) > 2 else ""
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) < len(hdr) or r[col["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[col["Kernel Name"]]
        unit = r[col["Metric Unit"]]
        v = float(r[col["Metric Value"]].replace(",", ""))
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
              "second": 1e3, "s": 1e3}.get(unit, 1.0)
        tot[name] += v
        cnt[name] += 1
    all_ms = sum(tot.values())
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none {note}, {sum(cnt.values())} launches")
    print("# cold-cache serialized launch times; compare shares, not absolutes")
    for name, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{100 * v / all_ms:6.2f}%  n={cnt[name]:4d}  {v:10.3f} ms  {name[:90]}")


if __name__ == "__main__":
    main()
