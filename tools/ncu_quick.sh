#!/bin/bash
# quick ncu of the boolean traversal kernel for each lib variant given as args
mkdir -p gpurun_out
for L in "$@"; do
  RSI_LIB=paper_2305_01867_b200/lib/$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trace -s 2 -c 1 -o gpurun_out/q_${L%.so} -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra-modes --mode ${MODE:-boolean} > /dev/null 2>&1
done
ls gpurun_out
