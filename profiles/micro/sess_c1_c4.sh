set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_client_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
for i in 1 2; do timeout 300 python profiles/micro/prof_c1.py 2>&1 | head -1; done
timeout 300 python profiles/micro/time_c4_ab.py 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:encode_ws -s 2 -c 1 -o gpurun_out/enc_head -f python profiles/micro/time_c4_ab.py > gpurun_out/ncu_enc_head.log 2>&1
tail -2 gpurun_out/ncu_enc_head.log
