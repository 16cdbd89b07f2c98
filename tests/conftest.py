import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run with -m gpu on a B200)")


class Case(dict):
    """One fixture case: dict of arrays with cloud()/camera() helpers."""

    def cloud(self, prefix=""):
        from paper_2604_12626_b200.cloud import GaussianCloud
        return GaussianCloud(self[prefix + "positions"], self[prefix + "sh_coeffs"], self[prefix + "opacities"],
                             self[prefix + "log_scales"], self[prefix + "rotations"])

    def camera(self, prefix="cam_"):
        from paper_2604_12626_b200.camera import Camera
        fx, fy, cx, cy, near, far = self[prefix + "intr"]
        w, h = (int(v) for v in self[prefix + "size"])
        return Camera(fx, fy, cx, cy, w, h, near, far, self[prefix + "w2c"])

    def background(self):
        bg = self["background"]
        return None if np.isnan(bg).any() else bg


def load_cases(name):
    data = np.load(os.path.join(GOLDEN, name + ".npz"))
    n = int(data["n_cases"])
    cases = [Case() for _ in range(n)]
    for key in data.files:
        if key == "n_cases":
            continue
        i, k = key.split("/", 1)
        cases[int(i)][k] = data[key]
    return cases


@pytest.fixture(scope="session")
def golden():
    return load_cases
