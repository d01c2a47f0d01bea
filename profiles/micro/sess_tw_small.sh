# two-pass 2^22 / 2^23 (twiddled 1024- / 2048-row column rings): parity tests,
# then the large-size timings with this tree's library and with alt/base.so
# (built before the change)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fft_gpu.py -q -x -k "two_pass or above_2e17 or large_in_place or ring_kernels or column_pass or 2d" > gpurun_out/tw_tests.log 2>&1; tail -3 gpurun_out/tw_tests.log
echo "== new"; timeout 300 python profiles/micro/time_large1d.py 2>&1 | head -4
echo "== old"; DPP_LIB_PATH=$PWD/alt/base.so timeout 300 python profiles/micro/time_large1d.py 2>&1 | head -4
