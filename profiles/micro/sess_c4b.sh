set -x
timeout 900 python -m pytest tests/test_imgc_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q -p no:cacheprovider -k "c4" 2>&1 | tail -3
bash profiles/micro/ab_c4.sh alt/head.so paper_1203_4938_b200/libdpp_b200.so
