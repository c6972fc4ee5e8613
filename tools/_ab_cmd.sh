#!/bin/bash
# scratch A/B driver (GPU box): rsi_test short head chunk per mode
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
rm -f gpurun_out/ab.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rsi_test or sparse or pycuda" > gpurun_out/ab.log 2>&1
for rep in 1 2; do for head in 0 262144 131072 65536; do
  RSI_TEST_HEAD=$head MODES=boolean,barycentric,intercept_count timeout 300 python tools/e2e_probe.py >> gpurun_out/ab.log 2>&1
done; done
RSI_TEST_HEAD=131072 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rsi_test or sparse or pycuda" >> gpurun_out/ab.log 2>&1
