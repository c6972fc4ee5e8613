#!/bin/bash
# scratch A/B driver (GPU box): early fetch of the nearest child's record (boolean)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python - <<'PY' >> gpurun_out/ab_build.log 2>&1
from paper_2305_01867_b200 import _build
_build.build_variant("qf1", {"RSI_QPF": 1})
_build.build_variant("qf0", {"RSI_QPF": 0})
PY
MODES=boolean bash tools/variants.sh "qf1 qf0 qf1 qf0" "sphere paper_terrain" > gpurun_out/ab.log 2>&1
