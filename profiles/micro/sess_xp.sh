set -x
timeout 900 python -m pytest tests/test_fft_gpu.py -q -p no:cacheprovider -x -k "numpy_f64 or two_pass or above_2e17 or in_place" 2>&1 | tail -4
cat > /tmp/one28.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_1203_4938_b200 import ops
n = 1 << int(sys.argv[1]); b = int(sys.argv[2])
x = torch.randn((b, n), dtype=torch.complex64, device='cuda'); y = torch.empty_like(x)
for _ in range(3): ops.fft_forward(x, n, out=y)
torch.cuda.synchronize()
PY
for m in "28 1" "24 4"; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python /tmp/one28.py $m 2>/dev/null | grep -v "^==" | tail -9 | cut -c1-250
DPP_LIB_PATH=$PWD/alt/head.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python /tmp/one28.py $m 2>/dev/null | grep -v "^==" | tail -12 | cut -c1-250
done
