for c in 16 8; do
for m in 5 7 9; do
  export DPP_FFT_CLUSTER_MODE=$m DPP_FFT_C65536=$c
  echo "C $c mode $m $(timeout 300 python -m pytest tests/test_fft_gpu.py -q -x -k 'every_size and 16 or batch_not' 2>&1 | tail -1) $(timeout 120 python profiles/micro/time_fft.py --iters 30)"
done
done
