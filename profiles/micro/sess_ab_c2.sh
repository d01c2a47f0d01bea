# A/B of C2 ring-kernel variants (alt/*.so, built by build_variant.py) against
# the shipped library: time + output digest, interleaved, two rounds
mkdir -p gpurun_out
for r in 1 2; do
  for lib in paper_1203_4938_b200/libdpp_b200.so "$@"; do
    DPP_LIB_PATH=$PWD/$lib timeout 120 python profiles/micro/ab_c2.py ${AB_ARGS:-} 2>&1 | tail -1
  done
done
