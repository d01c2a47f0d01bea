"""GPU k-means on the C4 frame's training blocks: per-kernel times under ncu
(run with ncu --metrics gpu__time_duration.sum), or wall time without."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1203_4938_b200 import kmeans as km  # noqa: E402
from paper_1203_4938_b200.apps import imgc  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
g = imgc.synthetic_image(side, side, seed=7)[..., 1]
px = torch.from_numpy(np.ascontiguousarray(g)).cuda()
norm64, grad = km.block_stats_device(px, 1, side, side)
keep = torch.nonzero(grad >= 1.0).squeeze(1)
train = norm64.index_select(0, keep)
torch.cuda.synchronize()
t0 = time.perf_counter()
tr = []
km.kmeans_device(train, 256, 0, trace=tr)
torch.cuda.synchronize()
print(f"n={train.shape[0]} kmeans {time.perf_counter() - t0:.4f} s, {len(tr)} Lloyd iterations", flush=True)
