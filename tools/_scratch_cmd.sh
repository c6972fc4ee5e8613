#!/bin/bash
# scratch A/B driver (GPU box): rsi_test pipeline (H2D streams x slots)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rsi_test or sparse or pycuda" > gpurun_out/ab.log 2>&1
for rep in 1 2; do
for cfg in "1 2" "2 4" "2 3" "1 4" "2 6"; do
  set -- $cfg
  RSI_TEST_H2D=$1 RSI_TEST_SLOTS=$2 timeout 300 python tools/e2e_probe.py >> gpurun_out/ab.log 2>&1
done; done
