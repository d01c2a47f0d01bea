"""Debug: fused pair calls (b x 4096^2): determinism, pair vs single schedule,
point symmetry, where the differences sit."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

from paper_1203_4938_b200 import ops
from paper_1203_4938_b200.apps import chain

b = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
g = torch.Generator(device="cuda").manual_seed(1)
imgs = torch.randint(0, 256, (b, rows, 4096), dtype=torch.uint8, device="cuda", generator=g)
out = torch.empty_like(imgs)
out2 = torch.empty_like(imgs)
assert ops.fft2d_u8_spectrum(imgs.reshape(-1), rows, 4096, chain.ALPHA, out.reshape(-1))
assert ops.fft2d_u8_spectrum(imgs.reshape(-1), rows, 4096, chain.ALPHA, out2.reshape(-1))
print("deterministic:", torch.equal(out, out2))
for i in range(b):
    one = torch.empty_like(imgs[i])
    assert ops.fft2d_u8_spectrum(imgs[i].reshape(-1), rows, 4096, chain.ALPHA, one.reshape(-1))
    d = (out[i].short() - one.short()).abs()
    bad = (d > 0).nonzero()
    print(f"image {i}: differ {bad.shape[0]}, max {int(d.max())}")
    if bad.shape[0]:
        r, c = bad[:, 0], bad[:, 1]
        print("  rows (first):", r[:12].tolist())
        print("  cols (first):", c[:12].tolist())
        print("  col hist mod 16:", torch.bincount(c % 16, minlength=16).tolist())
        print("  col<2048:", int((c < 2048).sum()), " col==0:", int((c == 0).sum()), " col==2048:", int((c == 2048).sum()))
        big = (d > 1).nonzero()[:8]
        for rr, cc in big.tolist():
            print("   ", rr, cc, int(out[i, rr, cc]), int(one[i - i, rr, cc] if False else one[rr, cc]))
    m = torch.roll(torch.flip(out[i], dims=(0, 1)), shifts=(1, 1), dims=(0, 1))
    print("  symmetric:", torch.equal(out[i], m), int((out[i] != m).sum()))
