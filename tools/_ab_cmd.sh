#!/bin/bash
# scratch A/B driver (GPU box): intercept_count two-hit fast path
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python - <<'PY' >> gpurun_out/ab_build.log 2>&1
from paper_2305_01867_b200 import _build
_build.build_variant("cp1", {"RSI_COUNT_PAIR": 1})
_build.build_variant("cp0", {"RSI_COUNT_PAIR": 0})
PY
MODES=intercept_count bash tools/variants.sh "cp1 cp0 cp1 cp0" "sphere terrain paper_terrain" > gpurun_out/ab.log 2>&1
