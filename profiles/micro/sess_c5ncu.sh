# ncu of the shipped C5 pair schedule: launch list + full capture of both passes
set -x
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python profiles/micro/c5_once.py 64 > /dev/null 2>&1; echo rc=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fft4096_ws -s 1 -c 1 -o gpurun_out/c5_rows -f python profiles/micro/c5_once.py 64 > /dev/null 2>&1; echo rc=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fft_cols_l2w -s 1 -c 1 -o gpurun_out/c5_cols -f python profiles/micro/c5_once.py 64 > /dev/null 2>&1; echo rc=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:encode_ws -s 1 -c 1 -o gpurun_out/c4_enc -f python profiles/micro/time_c4_ab.py > /dev/null 2>&1; echo rc=$?
