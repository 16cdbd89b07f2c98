"""Prints an ncu launch list (--metrics gpu__time_duration.sum[,launch__grid_size] --csv) as one line
per launch: id, kernel, grid, microseconds; then the total."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID") 
hdr = rows[start]
kn, mn, mv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
data, order = {}, []
for r in rows[start + 1:]:
    k = (r[0], r[kn])
    if k not in data:
        data[k] = {}
        order.append(k)
    data[k][r[mn]] = r[mv].replace(",", "")
tot = 0.0
for k in order:
    d = data[k]
    us = float(d.get("gpu__time_duration.sum", 0)) / 1e3
    tot += us
    print(f"{k[0]:>4} {k[1].split('(')[0][-48:]:>48} grid {d.get('launch__grid_size', '-'):>8} {us:10.1f} us")
print(f"total {tot / 1e3:.2f} ms over {len(order)} launches")
