#!/bin/bash
# Round-end refresh of the bench lines and the C3 launch list under gpurun_out/.
# usage (on the GPU box): bash tools/refresh_profiles.sh <tag>
tag=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; tail -1 gpurun_out/${tag}_gpu_tests.log
for wl in c3 c4 c5; do
  python bench.py --workload $wl > gpurun_out/${tag}_bench_$wl.json 2> gpurun_out/${tag}_bench_$wl.err || echo "bench $wl failed"
done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err
python tools/one_frame.py c3 1 > /dev/null && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c3.csv \
      python tools/one_frame.py c3 1 > gpurun_out/${tag}_ncu_launch.log 2>&1
python tools/launches.py gpurun_out/${tag}_launches_c3.csv 25 > gpurun_out/${tag}_launches_c3.txt
for f in gpurun_out/${tag}_bench_*.json; do echo "$f: $(tail -c 300 $f | head -c 300)"; done
