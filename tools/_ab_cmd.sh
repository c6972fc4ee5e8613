#!/bin/bash
# scratch A/B driver (GPU box): rsi_test with odd chunks on a second handle / stream
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ab.log 2>&1
tail -1 gpurun_out/ab.log > gpurun_out/ab2.log
for rep in 1 2; do for d in 0 1; do
  RSI_TEST_DUAL=$d MODES=boolean,barycentric,intercept_count timeout 300 python tools/e2e_probe.py >> gpurun_out/ab2.log 2>&1
done; done
