"""Asset ingest measurement: a 1M-gaussian degree-3 PLY through
assets.load_gaussian_ply (file -> pinned host -> device unpack + validation) against the numpy
restatement of the reference's loader (oracle.load_gaussian_ply_numpy) on the host; the unpack
kernel alone is timed with CUDA events and put against the HBM copy peak. Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import oracle as O
from paper_2604_12626_b200 import _native as N
from paper_2604_12626_b200 import assets as A

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
path = "/tmp/bench_scene_deg3.ply"
rng = np.random.default_rng(0)
names = ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2"] + [f"f_rest_{i}" for i in range(45)] + \
        ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
table = rng.normal(size=(n, len(names))).astype("<f4")
with open(path, "wb") as f:
    f.write(("ply\nformat binary_little_endian 1.0\n" + f"element vertex {n}\n" +
             "".join(f"property float {p}\n" for p in names) + "end_header\n").encode("ascii"))
    f.write(table.tobytes())
file_bytes = os.path.getsize(path)

# CPU: the reference loader's numpy path (warm page cache: read once first)
O.load_gaussian_ply_numpy(path)
t0 = time.perf_counter()
ref = O.load_gaussian_ply_numpy(path)
cpu_s = time.perf_counter() - t0

# GPU end to end through the public loader
torch.cuda.synchronize()
A.load_gaussian_ply(path)
torch.cuda.synchronize()
t0 = time.perf_counter()
dc = A.load_gaussian_ply(path)
torch.cuda.synchronize()
e2e_s = time.perf_counter() - t0
pos, sh, op, ls, rot = dc.to_host()
exact = all(np.array_equal(a, b) for a, b in zip((pos, sh, op, ls, rot), ref))

# the unpack kernel alone (device-resident table), CUDA events
tab, cols, k = A.read_ply_table(path)
t = torch.from_numpy(np.ascontiguousarray(tab)).cuda()
outs = [torch.empty((n, 4), device="cuda") for _ in range(3)] + [torch.empty((k * 3, n), device="cuda")]
flags = torch.zeros(n, dtype=torch.uint8, device="cuda")
cnt = torch.zeros(10, dtype=torch.int64, device="cuda")
lib = N.load()
import ctypes


def run():
    N.check(lib.sn_unpack_ply(n, tab.shape[1], t.data_ptr(), cols.ctypes.data_as(ctypes.c_void_p), k,
                              outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(), outs[3].data_ptr(),
                              flags.data_ptr(), cnt.data_ptr(), torch.cuda.current_stream().cuda_stream))


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 20
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
kms = e0.elapsed_time(e1) / reps
alg = n * len(names) * 4 + n * (3 * 16 + 3 * k * 4) + n  # table read + buffers + flags written
try:
    peak = float(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    peak = 6650.0
print(json.dumps({
    "metric": "3DGS PLY ingest (1M gaussians, SH degree 3) to the device layout", "n_gaussians": n,
    "file_bytes": file_bytes, "bit_exact_vs_reference_loader": bool(exact),
    "gpu_e2e_s": e2e_s, "gpu_e2e_gaussians_per_s": n / e2e_s,
    "cpu_reference_port_s": cpu_s, "cpu_cores": 1, "speedup_e2e": cpu_s / e2e_s,
    "unpack_kernel_ms": kms, "unpack_roofline": {"bound": "hbm", "achieved": alg / kms / 1e6, "peak": peak,
                                                 "unit": "GB/s", "frac": alg / kms / 1e6 / peak,
                                                 "alg_bytes": alg}}))
