# (session-5 record: alt/old30.so was built from the previous commit's fft_large.cu with build_variant.py)
# two-pass 2^30 (32768 x 32768: twiddled 32768-row ring): parity tests, then
# large-size timings with this tree's library and alt/old30.so (pre-change dispatch)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_fft_gpu.py -q -x -k "two_pass or above_2e17 or large_in_place or 2d or column" > gpurun_out/tw30_tests.log 2>&1; tail -3 gpurun_out/tw30_tests.log
echo "== new"; timeout 300 python profiles/micro/time_large1d.py 2>&1 | tail -3
echo "== old"; DPP_LIB_PATH=$PWD/alt/old30.so timeout 300 python profiles/micro/time_large1d.py 2>&1 | tail -3
