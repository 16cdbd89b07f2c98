"""Small renders for compute-sanitizer (memcheck / racecheck / synccheck): BASELINE config 0 (scene
only, 256x256, 20k gaussians) and a 2-avatar 160x120 batch of 3 envs through both binners, the
float64 exact mode and the observation payload. Prints 'sanitize cases ok' on success."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_12626_b200 import renderer as R  # noqa: E402
from paper_2604_12626_b200 import synthetic as S  # noqa: E402
from paper_2604_12626_b200.batch import BatchRenderer  # noqa: E402


def main():
    scene, cam = S.config0()
    R.render_frames(scene, [cam], np.zeros(3), contrib=True)
    box = S.room_box(1_000_000)
    bundles = [S.make_avatar(2000, seed=60 + i, n_frames=8, floor_lo=(3.0, 3.0), floor_hi=(5.0, 5.0)) for i in range(2)]
    room = S.make_scene(20_000, box[0], box[1], seed=61)
    cams = S.room_cameras(3, box, seed=62, width=160, height=120)
    br = BatchRenderer(room, bundles, start_offsets=[0.0, 0.1], background=(0.5, 0.5, 0.5))
    times = np.array([0.0, 0.1, 0.2])
    for exact in (False, True):
        for binning in (-1, 1):
            br.render(cams, times, contrib=True, stats=True, exact=exact, payload=True, binning=binning)
    R.device_tiles(80, 0, 1, context=br.context)
    R.device_tiles(80, 1, 1, context=br.context)
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
