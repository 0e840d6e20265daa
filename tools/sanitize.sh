#!/bin/bash
# compute-sanitizer evidence for the shared-memory / mbarrier / TMA / DSMEM
# kernels: racecheck and synccheck on the hot kernels, memcheck on
# whole frames. Logs land in gpurun_out/<tag>_sanitize_<tool>.txt.
# usage (GPU box): bash tools/sanitize.sh <tag>
tag=${1:-rXX}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool extra-args precision
  timeout 1500 $CS --tool $1 $2 --print-limit 50 python tools/sanitize_run.py $3 \
      > gpurun_out/${tag}_sanitize_$1_$3.txt 2>&1
  echo "$1 $3 rc=$?" >> gpurun_out/${tag}_sanitize_summary.txt
  tail -3 gpurun_out/${tag}_sanitize_$1_$3.txt >> gpurun_out/${tag}_sanitize_summary.txt
}
: > gpurun_out/${tag}_sanitize_summary.txt
run memcheck "--leak-check no" both
run racecheck "--racecheck-report all" fp32
run racecheck "--racecheck-report all" fp64
run synccheck "" both
cat gpurun_out/${tag}_sanitize_summary.txt
