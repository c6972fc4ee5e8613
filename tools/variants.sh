#!/bin/bash
# GPU-box helper: parity subset + timing for each variant library.
# Usage (under gpurun): bash tools/variants.sh "base bf0 pf" [workloads]
vars=${1:-base}
wls=${2:-"sphere paper_terrain"}
mkdir -p gpurun_out
for v in $vars; do
  L=paper_2305_01867_b200/lib/librsi_$v.so
  RSI_LIB=$L timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sphere or terrain or vertices or stacked or single" 2>&1 | tail -1 | sed "s/^/[$v parity] /"
  for wl in $wls; do
    for rep in 1 2; do
      RSI_LIB=$L WL=$wl COUNTERS=0 timeout 300 python tools/sweep.py 2>&1 | sed "s/^/[$wl r$rep] /"
    done
  done
done
