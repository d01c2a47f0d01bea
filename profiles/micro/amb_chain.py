"""Ambiguous-block fraction of the TC encoder on C5 spectrum images vs C4 noise images."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def run(img, cb, dev):
    import torch
    from paper_1203_4938_b200 import _lib
    h, w = img.shape
    nb = (h // 4) * (w // 4)
    rec = torch.empty(nb * 3, dtype=torch.uint8, device=dev)
    cbp = torch.empty(nb, dtype=torch.uint8, device=dev)
    crp = torch.empty(nb, dtype=torch.uint8, device=dev)
    amb = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().dpp_imgc_encode_tc_debug(img.data_ptr(), 1, h, w, cb.data_ptr(), 256, rec.data_ptr(),
                                                    cbp.data_ptr(), crp.data_ptr(), ctypes.c_float(1.0),
                                                    amb.data_ptr(), None))
    sig = rec.view(-1, 3)[:, 1]
    return int(amb.item()) / nb, float((sig == 0).float().mean())


def main():
    import torch
    from paper_1203_4938_b200 import ops
    from paper_1203_4938_b200.apps import chain
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    img = torch.randint(0, 256, (4096, 4096), dtype=torch.uint8, device=dev, generator=g)
    cb = torch.randn((256, 16), device=dev, generator=g)
    cb = (cb - cb.mean(-1, keepdim=True)) / cb.std(-1, unbiased=False, keepdim=True)
    z = torch.empty((4096, 4096), dtype=torch.complex64, device=dev)
    ops.u8_to_complex(img.reshape(-1), torch.view_as_real(z).reshape(-1))
    ops.fft2d_forward(z, 4096, 4096, out=z)
    spec = torch.empty((4096, 4096), dtype=torch.uint8, device=dev)
    ops.spectrum_u8(torch.view_as_real(z).reshape(-1), spec.reshape(-1), chain.ALPHA)
    print("noise image: ambiguous %.4f, sigma_idx==0 %.4f" % run(img, cb, dev))
    print("spectrum image: ambiguous %.4f, sigma_idx==0 %.4f" % run(spec, cb, dev))
    vals, counts = torch.unique(spec, return_counts=True)
    print("spectrum histogram top:", sorted(zip(counts.tolist(), vals.tolist()))[-5:])


if __name__ == "__main__":
    main()
