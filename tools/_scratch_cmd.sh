#!/bin/bash
# scratch A/B driver (GPU box): approximate reciprocal in the MT hit path + fast |d|
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ab_pytest.log 2>&1
tail -2 gpurun_out/ab_pytest.log > gpurun_out/ab.log
python - <<'PY' >> gpurun_out/ab_build.log 2>&1
from paper_2305_01867_b200 import _build
_build.build_variant("mr1", {"RSI_MT_RCP": 1, "RSI_FAST_NORM": 1})
_build.build_variant("mr0", {"RSI_MT_RCP": 0, "RSI_FAST_NORM": 0})
PY
MODES=barycentric,intercept_count bash tools/variants.sh "mr1 mr0 mr1 mr0" "sphere paper_terrain terrain" >> gpurun_out/ab.log 2>&1
timeout 1200 python tools/parity_full.py > gpurun_out/parity_full_mr.json 2>&1
