set -x
timeout 120 compute-sanitizer --tool memcheck --show-backtrace no python profiles/micro/time_c4_ab.py 2>&1 | tail -3
timeout 120 python profiles/micro/time_c4_ab.py 2>&1 | tail -1
DPP_LIB_PATH=$PWD/alt/head.so timeout 120 python profiles/micro/time_c4_ab.py 2>&1 | tail -1
timeout 120 python profiles/micro/time_c4_ab.py 2>&1 | tail -1
DPP_LIB_PATH=$PWD/alt/head.so timeout 120 python profiles/micro/time_c4_ab.py 2>&1 | tail -1
timeout 400 python -m pytest tests/test_imgc_gpu.py tests/test_fullsize_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 300 python profiles/micro/time_c5_parts.py 64
