# round-2 evidence: bench line, launch list of the same command under ncu
# (cold-cache, serialised: shares only), one --set full capture of the C2 kernel
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/bench_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft65536_l2w -s 2 -c 1 -o gpurun_out/c2_full -f python profiles/drive.py fft --iters 3 > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
tail -c 3000 gpurun_out/bench.json
