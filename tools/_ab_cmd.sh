#!/bin/bash
# scratch A/B driver (GPU box): rsi_test tail schedule (halving final chunks) per mode
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
rm -f gpurun_out/ab.log
for rep in 1 2; do for tail in 0 262144 131072 65536; do
  RSI_TEST_TAIL=$tail MODES=boolean,barycentric,intercept_count timeout 300 python tools/e2e_probe.py >> gpurun_out/ab.log 2>&1
done; done
