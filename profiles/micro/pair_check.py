import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1203_4938_b200 import ops
from oracle import fft_oracle as fo
dev = torch.device('cuda:0')
for batch in (1, 2, 3, 5, 148, 333):
    rng = np.random.default_rng(batch)
    x = (rng.standard_normal((batch, 65536)) + 1j*rng.standard_normal((batch, 65536))).astype(np.complex64)
    y = ops.fft_forward(torch.from_numpy(x).to(dev), 65536).cpu().numpy()
    rows = [0, batch-1, batch//2]
    err = max(np.linalg.norm(y[r]-fo.fft(x[r]))/np.linalg.norm(fo.fft(x[r])) for r in rows)
    print('batch', batch, 'err', err, flush=True)
