"""C4 encoder timing on the SURVEY §8(d) frame (A/B helper).

    python profiles/micro/time_encode.py

synthetic_image(8192, 8192, seed=7) green channel as gray, the reference-trained
codebook (tests/golden/c4_golden.npz); prints ms per frame, the fraction of
blocks that needed the exact re-check, and whether the bitstream SHA-256
equals the reference's.
"""

import ctypes
import hashlib
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_1203_4938_b200 import _lib, ops  # noqa: E402
from paper_1203_4938_b200.apps.imgc import CompressedImage, synthetic_image  # noqa: E402

dev = torch.device("cuda:0")
gold = np.load(ROOT / "tests/golden/c4_golden.npz")
h = w = 8192
g = synthetic_image(w, h, seed=7)[..., 1].copy()
img = torch.from_numpy(g).to(dev)
cb = torch.from_numpy(gold["codebook"]).to(dev)
nb = (h // 4) * (w // 4)
rec = torch.empty(nb * 3, dtype=torch.uint8, device=dev)
cbp = torch.empty(nb, dtype=torch.uint8, device=dev)
crp = torch.empty(nb, dtype=torch.uint8, device=dev)
for _ in range(3):
    ops.encode(img, 1, h, w, cb, rec, cbp, crp)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    ops.encode(img, 1, h, w, cb, rec, cbp, crp)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
blob = CompressedImage.from_records(w, h, gold["codebook"], rec.cpu().numpy(), cbp.cpu().numpy(),
                                    crp.cpu().numpy()).to_bytes()
amb = torch.zeros(1, dtype=torch.int64, device=dev)
lib = _lib.load()
lib.dpp_imgc_encode_tc_debug(ctypes.c_void_p(img.data_ptr()), 1, h, w, ctypes.c_void_p(cb.data_ptr()), 256,
                             ctypes.c_void_p(rec.data_ptr()), ctypes.c_void_p(cbp.data_ptr()),
                             ctypes.c_void_p(crp.data_ptr()), ctypes.c_float(1.0), ctypes.c_void_p(amb.data_ptr()),
                             None)
torch.cuda.synchronize()
print(f"C4 encode {ms:.4f} ms/frame = {h * w / ms / 1e6:.0f} GPixel/s; exact re-check {int(amb.item())} of {nb} "
      f"blocks ({100 * int(amb.item()) / nb:.3f} %); bitstream == reference: "
      f"{hashlib.sha256(blob).hexdigest() == str(gold['blob_sha'])}")
