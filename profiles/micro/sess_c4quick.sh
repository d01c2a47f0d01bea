set -x
timeout 120 python profiles/micro/time_c4_ab.py 2>&1 | tail -1
timeout 300 python -m pytest tests/test_imgc_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -2
DPP_LIB_PATH=$PWD/alt/head.so timeout 120 python profiles/micro/time_c4_ab.py 2>&1 | tail -1
timeout 120 python profiles/micro/time_c4_ab.py 2>&1 | tail -1
