#!/bin/bash
# scratch A/B driver (GPU box): intercept_count at 6 CTAs / SM (more registers, no spills)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python - <<'PY' >> gpurun_out/ab_build.log 2>&1
from paper_2305_01867_b200 import _build
_build.build_variant("c7", {"RSI_COUNT_MINB": 7})
_build.build_variant("c6", {"RSI_COUNT_MINB": 6})
PY
MODES=intercept_count bash tools/variants.sh "c7 c6 c7 c6" "sphere terrain paper_terrain" > gpurun_out/ab.log 2>&1
