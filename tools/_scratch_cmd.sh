#!/bin/bash
# scratch A/B driver (GPU box): intercept_count at 8 CTAs / SM (64 registers)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python - <<'PY' >> gpurun_out/ab_build.log 2>&1
from paper_2305_01867_b200 import _build
_build.build_variant("cm7", {"RSI_COUNT_MINB": 7})
_build.build_variant("cm8", {"RSI_COUNT_MINB": 8})
PY
MODES=intercept_count bash tools/variants.sh "cm7 cm8 cm7 cm8" "sphere terrain paper_terrain" > gpurun_out/ab.log 2>&1
