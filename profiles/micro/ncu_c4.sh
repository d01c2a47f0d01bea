ncu --set full --clock-control none --import-source on -k regex:encode_ws -s 2 -c 1 -o gpurun_out/enc_cur -f python profiles/micro/time_c4_ab.py > gpurun_out/ncu_enc_cur.log 2>&1
tail -2 gpurun_out/ncu_enc_cur.log
