#!/bin/bash
# GPU-box helper: full GPU tests on the default lib, then parity subset +
# min_trav sweep per variant.  Usage: bash tools/variants2.sh "v1 v2" "8:1,16:1,24:1"
vars=${1:-base}
cfgs=${2:--1:1}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in $vars; do
  L=paper_2305_01867_b200/lib/librsi_$v.so
  RSI_LIB=$L timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sphere or terrain or vertices or stacked or single or scaled" 2>&1 | tail -1 | sed "s/^/[$v parity] /"
  for wl in sphere paper_terrain; do
    RSI_LIB=$L WL=$wl CFGS=$cfgs COUNTERS=${COUNTERS:-0} timeout 600 python tools/sweep.py 2>&1 | sed "s/^/[$wl] /"
  done
done
