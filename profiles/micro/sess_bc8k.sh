echo "== shipped"; timeout 300 python profiles/micro/time_large1d.py 2>&1 | sed -n 6,8p
echo "== bc 8192"; DPP_LIB_PATH=$PWD/alt/bc8k.so timeout 300 python profiles/micro/time_large1d.py 2>&1 | sed -n 6,8p
DPP_LIB_PATH=$PWD/alt/bc8k.so timeout 300 python -c "
import torch, numpy as np
from paper_1203_4938_b200 import ops
n = 1 << 26
x = torch.randn(n, dtype=torch.complex64, device='cuda')
y = ops.fft_forward(x, n).cpu().numpy()
r = np.fft.fft(x.cpu().numpy().astype(np.complex128))
print('bc8k 2^26 rel_l2', float(np.linalg.norm(y - r) / np.linalg.norm(r)))
"
