#!/bin/bash
# scratch A/B driver (GPU box): rsi_test chunk size per mode
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
rm -f gpurun_out/ab.log
for rep in 1 2; do for ch in 1048576 524288 393216 262144; do
  RSI_TEST_CHUNK=$ch MODES=boolean,barycentric,intercept_count timeout 300 python tools/e2e_probe.py >> gpurun_out/ab.log 2>&1
done; done
