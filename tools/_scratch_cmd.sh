#!/bin/bash
# scratch A/B driver (GPU box): branch-free ray setup
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python - <<'PY' >> gpurun_out/ab_build.log 2>&1
from paper_2305_01867_b200 import _build
_build.build_variant("sbf1", {"RSI_SLAB_BF": 1})
_build.build_variant("sbf0", {"RSI_SLAB_BF": 0})
PY
bash tools/variants.sh "sbf1 sbf0 sbf1 sbf0" "sphere paper_terrain" > gpurun_out/ab.log 2>&1
