set -x
timeout 200 python profiles/micro/dbg_pair.py 3 4096 2>&1 | tail -30
timeout 200 python profiles/micro/dbg_pair.py 2 16384 2>&1 | tail -30
timeout 600 python -m pytest tests/test_chain_gpu.py tests/test_fullsize_gpu.py -k "c5 or fused or chain" -q -s -p no:cacheprovider 2>&1 | grep -v "^frame" | tail -40
