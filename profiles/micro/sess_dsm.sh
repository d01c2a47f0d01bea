set -x
for b in 1 7 64 4096; do
  timeout 120 python profiles/micro/ab_dsm.py $b
  DPP_FFT_DSM=3 timeout 120 python profiles/micro/ab_dsm.py $b
  DPP_FFT_DSM=2 timeout 120 python profiles/micro/ab_dsm.py $b
done
