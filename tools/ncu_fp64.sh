#!/bin/bash
# ncu --set full captures of the float64 path's top kernels at the C3 finest
# level (LEVELS=1: the 1024^2 level alone), raw pages exported as CSV.
# usage (on the GPU box): bash tools/ncu_fp64.sh <tag> [pd-kernel-regex]
tag=${1:-rXX}
pd=${2:-k64_block}
mkdir -p gpurun_out
LEVELS=1 python tools/one_frame64.py c3 1 > /dev/null || exit 1
cap() {  # name regex skip
  LEVELS=1 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$2" --launch-skip $3 -c 1 -o gpurun_out/${tag}_$1 -f \
      python tools/one_frame64.py c3 1 > gpurun_out/${tag}_$1.log 2>&1
  ncu -i gpurun_out/${tag}_$1.ncu-rep --page raw --csv > gpurun_out/${tag}_$1_raw.csv 2>&1
  ncu -i gpurun_out/${tag}_$1.ncu-rep --page source --csv > gpurun_out/${tag}_$1_src.csv 2>&1
}
cap pd64 "$pd" 12
cap sample64 "k64_sample" 6
cap lin64 "k64_linearize" 6
ls -la gpurun_out/${tag}_*
