#!/bin/bash
# GPU-box helper: per-kernel roofline CSVs for the bench step (N_t = 1e4) and
# the N_t = 1e6 per-GPU share of configs[4].  Usage: bash tools/kernel_roofline.sh <tag>
tag=${1:-r1}
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_fp32_pred_on.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum
for m in boolean barycentric intercept_count; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/kr_${m}_${tag}.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra-modes --no-configs --mode $m > /dev/null 2>&1
done
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/kr_sphere1m_${tag}.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra-modes --no-configs --workload sphere1m --rays-per-gpu 12500000 > /dev/null 2>&1
ls gpurun_out/kr_*
