#!/bin/bash
# One `ncu --set full` capture per top kernel of a C3 frame (in-solve launches
# at the finest level), raw pages exported as CSV for summarising here.
# usage (on the GPU box): bash tools/ncu_full.sh <tag>
tag=${1:-rXX}
mkdir -p gpurun_out
python tools/one_frame.py c3 1 > /dev/null || exit 1
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$2" --launch-skip $3 -c 1 -o gpurun_out/${tag}_$1 -f \
      python tools/one_frame.py c3 1 > gpurun_out/${tag}_$1.log 2>&1
  ncu -i gpurun_out/${tag}_$1.ncu-rep --page raw --csv > gpurun_out/${tag}_$1_raw.csv 2>&1
}
# skip into the 1024^2 warp loop: <5,..> PD runs at 512^2 (launches 0..49) then 1024^2;
# k_sample_px<6> at 512^2 then 1024^2; k_iu_px at 256^2, 512^2, 1024^2
cap pd_fin "k_pd_tma<.int.5, .bool.0, .bool.1" 70
cap pd_lin "k_pd_tma<.int.5, .bool.1, .bool.0" 70
cap sample "k_sample_px<.int.6>" 70
cap iu "k_iu_px" 120
ls -la gpurun_out/${tag}_*
