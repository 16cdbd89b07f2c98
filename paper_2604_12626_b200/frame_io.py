"""Frame export from device frames (reference: splatnav/frame_io.py:11-58).

The quantization (uint8 colour, fp16 depth) and the PFM row flip run on the device
(sn_quantize_frames, sn_flip_rows); only the finished bytes cross PCIe. The file formats are the
reference's: 8-bit RGB PNG of clip(x, 0, 1) * 255 + 0.5 truncated (:11-15), grayscale
little-endian PFM with scale -1.0 and rows bottom-to-top (:23-31), raw float32 + JSON sidecar
(:45-51). Host arrays are accepted too (they are uploaded first).
"""

import json

import numpy as np
import torch

from . import _native as N


def _dev(x):
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x.contiguous().float()
    return torch.as_tensor(np.asarray(x, dtype=np.float32)).cuda()


def quantize(color, depth=None):
    """Device frames (...,3) float colour and (...) depth -> uint8 RGB and fp16 depth (device)."""
    c = _dev(color)
    npix = c.numel() // 3
    rgb = torch.empty(c.shape, dtype=torch.uint8, device=c.device)
    d16 = None
    d = None
    if depth is not None:
        d = _dev(depth)
        if d.numel() != npix:
            raise ValueError(f"depth has {d.numel()} pixels, colour {npix}")
        d16 = torch.empty(d.shape, dtype=torch.float16, device=c.device)
    N.check(N.load().sn_quantize_frames(npix, c.data_ptr(), d.data_ptr() if d is not None else None, rgb.data_ptr(),
                                        d16.data_ptr() if d16 is not None else None,
                                        torch.cuda.current_stream(c.device).cuda_stream))
    return rgb, d16


def save_color_png(color, path):
    """frame_io.save_color_png: (H, W, 3) colour in [0, 1] -> 8-bit PNG (quantized on the device)."""
    from PIL import Image
    rgb, _ = quantize(color)
    Image.fromarray(rgb.cpu().numpy(), mode="RGB").save(path)


def flip_rows(depth):
    """(..., H, W) device frames with their rows in reverse order (the PFM layout)."""
    d = _dev(depth)
    h, w = d.shape[-2], d.shape[-1]
    out = torch.empty_like(d)
    N.check(N.load().sn_flip_rows(d.numel() // (h * w), h, w, d.data_ptr(), out.data_ptr(),
                                  torch.cuda.current_stream(d.device).cuda_stream))
    return out


def save_depth_pfm(depth, path):
    """frame_io.save_depth_pfm: grayscale PFM, little-endian float32 (scale -1.0), bottom-to-top."""
    d = _dev(depth)
    h, w = d.shape
    data = flip_rows(d).cpu().numpy().astype("<f4")
    with open(path, "wb") as f:
        f.write(b"Pf\n")
        f.write(f"{w} {h}\n".encode("ascii"))
        f.write(b"-1.0\n")
        f.write(data.tobytes())


def save_depth_f32(depth, path, far):
    """frame_io.save_depth_f32: raw little-endian float32 plus a JSON sidecar."""
    d = _dev(depth)
    h, w = d.shape
    d.cpu().numpy().astype("<f4").tofile(path)
    with open(str(path) + ".json", "w", encoding="utf-8") as f:
        json.dump({"width": w, "height": h, "far": far}, f)
