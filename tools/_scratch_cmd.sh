#!/bin/bash
# scratch A/B driver (GPU box): predicated pop in the visit
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python - <<'PY' >> gpurun_out/ab_build.log 2>&1
from paper_2305_01867_b200 import _build
_build.build_variant("pp1", {"RSI_POP_PRED": 1})
_build.build_variant("pp0", {"RSI_POP_PRED": 0})
PY
bash tools/variants.sh "pp1 pp0 pp1 pp0" "sphere paper_terrain" > gpurun_out/ab.log 2>&1
