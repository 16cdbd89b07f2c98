"""Extract per-launch DRAM traffic of the bench's kernels from an `ncu --set full` report into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic) and print a summary.

usage: python scripts/ncu_traffic.py gpurun_out/prof_full.ncu-rep [out.json] [workload tag]
(the tag is bench.workload_tag of the profiled command; default: bench.py's default workload)
"""
import csv
import io
import json
import subprocess
import sys

STAGE_OF = {"blend_kernel<0, 0>": "scene.blend", "blend_kernel_lp2": "layer.blend",
            "scene_emit_kernel": "scene.emit", "scene_count_kernel": "scene.count",
            "fixup_kernel<0>": "scene.fixup", "fixup_kernel<2>": "layer.fixup"}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
           "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread"]


def main():
    rep = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_traffic.json"
    sys.path.insert(0, ".")
    import bench
    tag = sys.argv[3] if len(sys.argv) > 3 else bench.workload_tag(bench.parse([]))
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    result = {"_workload": tag}
    for r in data:
        name = r[col["Kernel Name"]]
        stage = next((v for k, v in STAGE_OF.items() if k in name), None)
        vals = {}
        for m in METRICS:
            if m in col and r[col[m]] not in ("", "n/a"):
                scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-3, "msecond": 1.0,
                         "nsecond": 1e-6}.get(units[col[m]], 1.0)
                vals[m] = float(r[col[m]].replace(",", "")) * scale
        print(f"== {name[:70]}")
        for m, v in vals.items():
            print(f"   {m:60s} {v:,.3f}")
        if stage and stage not in result:
            result[stage] = {"dram_bytes_per_launch": vals.get("dram__bytes_read.sum", 0.0) +
                             vals.get("dram__bytes_write.sum", 0.0),
                             "launches_per_step": 1, "source": f"ncu --set full ({rep.split('/')[-1]})",
                             "ncu_ms": vals.get("gpu__time_duration.sum"),
                             "warp_inst_per_launch": vals.get("smsp__inst_executed.sum"),
                             "issue_active_pct": vals.get("smsp__issue_active.avg.pct_of_peak_sustained_active")}
    with open(out, "w") as f:
        json.dump(result, f, indent=1)


if __name__ == "__main__":
    main()
