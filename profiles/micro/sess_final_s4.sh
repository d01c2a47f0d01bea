# session-4 closing run: full GPU suite, smoke, bench line, ncu --set full of
# the f16 encoder (pipe breakdown for r2_c4_notes.md)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:encode_ws -s 2 -c 1 -o gpurun_out/enc_f16 -f python profiles/micro/time_c4_ab.py > gpurun_out/ncu_enc_f16.log 2>&1; echo "ncu enc rc=$?"
tail -c 2500 gpurun_out/bench.json
