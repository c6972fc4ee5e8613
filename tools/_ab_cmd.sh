#!/bin/bash
# scratch A/B driver (GPU box): L1 prefetch of the chunk's next segments
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python - <<'PY' >> gpurun_out/ab_build.log 2>&1
from paper_2305_01867_b200 import _build
_build.build_variant("pl1", {"RSI_RAY_PF_L1": 1})
_build.build_variant("pl0", {"RSI_RAY_PF_L1": 0})
PY
bash tools/variants.sh "pl1 pl0 pl1 pl0" "sphere paper_terrain" > gpurun_out/ab.log 2>&1
