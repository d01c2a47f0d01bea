# A/B the DSMEM exchange variants of fft_cluster_kernel (DPP_FFT_CLUSTER_MODE), optional cluster size
mkdir -p gpurun_out
for m in ${MODES:-4 5}; do
 for c in ${CS:-8}; do
  export DPP_FFT_CLUSTER_MODE=$m DPP_FFT_C65536=$c
  tag=${m}_c$c
  timeout 300 python -m pytest tests/test_fft_gpu.py -q -k "every_size or golden or large" 2>&1 | tail -1 > gpurun_out/modes_$tag.log
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | cut -c1-160 >> gpurun_out/modes_$tag.log
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:fft_cluster -s 1 -c 1 -o gpurun_out/fft_mode$tag python profiles/drive.py fft --iters 2 > /dev/null 2>&1
 done
done
tail -n 3 gpurun_out/modes_*_c*.log
