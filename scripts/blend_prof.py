"""Diagnostic (library built with -DSN_BLEND_PROF, SPLATNAV_B200_LIB pointing at it): the scene
blend's walk counters on the bench workload -- warp iterations, boundary-band iterations, and
iterations where no pixel of the warp's 8 x 8 block lies inside the splat's support."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12626_b200 import _native as N
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer

lib = ctypes.CDLL(N.LIB_PATH)
hist = (ctypes.c_ulonglong * 16)()
n = 1_000_000
box = S.room_box(n)
scene = S.make_scene(n, box[0], box[1], seed=0)
br = BatchRenderer(scene, None, background=(1, 1, 1))
cams = S.room_cameras(64, box, seed=10_000)
ns = int(os.environ.get("NS", "-1"))
print("rendering", flush=True)
br.render(cams, views=False, near_slice=ns)
torch.cuda.synchronize()
print("warm", flush=True)
if hasattr(lib, "sn_debug_blend_prof"):
  lib.sn_debug_blend_prof(hist, 1)
  br.render(cams, views=False, near_slice=ns)
  torch.cuda.synchronize()
  lib.sn_debug_blend_prof(hist, 1)
  h = list(hist)
  print(f"warp iterations {h[0]}, boundary-band {h[1]} ({h[1] / max(h[0], 1):.4f}), no pixel inside {h[3]} "
      f"({h[3] / max(h[0], 1):.4f})")

if hasattr(lib, "sn_debug_fix_prof"):
    fx = (ctypes.c_ulonglong * 16)()
    lib.sn_debug_fix_prof(fx, 1)
    br.render(cams, views=False, near_slice=ns)
    torch.cuda.synchronize()
    lib.sn_debug_fix_prof(fx, 1)
    f = list(fx)
    print(f"deferred pixels {f[0]}: err > T/16 {f[1]}, T >= 1e-4(1+1e-6) {f[2]}, T within 1e-6 rel {f[3]}, "
          f"T below {f[4]}, forced {f[13]}, |T - 1e-4| <= 1e-9 {f[14]}, <= 4 contributions {f[15]}")
    print("log10(err / T) bins [<-7, -7, -6, -5, -4, -3, -2, >=-1]:", f[5:13])
