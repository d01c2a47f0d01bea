# C5 pair schedule: parity tests, then timing of the fused pass and the chain
set -x
mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool memcheck --show-backtrace no python profiles/micro/dbg_pair.py 3 2>&1 | tail -8
timeout 600 python -m pytest tests/test_chain_gpu.py tests/test_fullsize_gpu.py -k "c5 or fused or chain" -q -s -p no:cacheprovider 2>&1 | tail -25
timeout 300 python profiles/micro/time_c5_parts.py 64
timeout 300 python profiles/micro/time_c5_parts.py 64
