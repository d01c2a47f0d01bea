# (records a session-5 A/B: alt/oldfft/fft.py was the pre-change apps/fft.py; the change was not kept)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fft_gpu.py -q -k pinned_host_pipeline > gpurun_out/e2e_test.log 2>&1; tail -2 gpurun_out/e2e_test.log
for r in 1 2; do
  timeout 120 python profiles/micro/time_e2e_chunks.py 128 2>&1 | tail -1
  cp paper_1203_4938_b200/apps/fft.py /tmp/new_fft.py; cp alt/oldfft/fft.py paper_1203_4938_b200/apps/fft.py
  echo -n "old: "; timeout 120 python profiles/micro/time_e2e_chunks.py 128 2>&1 | tail -1
  cp /tmp/new_fft.py paper_1203_4938_b200/apps/fft.py
done
