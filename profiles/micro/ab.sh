#!/bin/bash
# A/B: time_fft.py (args "$@") with alt/head.so and the working-tree library, twice each, interleaved
for r in 1 2; do
  for lib in alt/head.so paper_1203_4938_b200/libdpp_b200.so; do
    echo "$lib: $(DPP_LIB_PATH=$PWD/$lib timeout 120 python profiles/micro/time_fft.py "$@" 2>&1 | tail -1)"
  done
done
