for r in 1 2; do
  for lib in "$@"; do
    DPP_LIB_PATH=$PWD/$lib timeout 300 python profiles/micro/time_c4_ab.py 2>&1 | tail -1
  done
done
