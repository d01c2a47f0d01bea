timeout 200 python profiles/micro/dbg_pair.py 3 4096 2>&1 | tail -14
for v in "" alt/c5_nostg.so; do DPP_LIB_PATH=$v timeout 120 python profiles/micro/time_c5_fft.py 64; done
timeout 600 python -m pytest tests/test_chain_gpu.py tests/test_fullsize_gpu.py -k "c5 or fused or chain" -q -s -p no:cacheprovider 2>&1 | grep -v "^frame" | tail -12
