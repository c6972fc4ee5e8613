#!/bin/bash
# GPU-box helper: launch list + full ncu captures of the traversal kernels.
# Usage (under gpurun): bash tools/profile.sh <tag>
tag=${1:-r1}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extra-modes --no-configs"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv $B > /dev/null 2>&1
for m in boolean barycentric intercept_count; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trace -s 2 -c 1 -o gpurun_out/prof_${m}_${tag} -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra-modes --no-configs --mode $m > /dev/null 2>&1
done
ls -la gpurun_out
