#!/bin/bash
# scratch A/B driver (GPU box): L2 prefetch of the chunk's next segments (boolean / barycentric)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python - <<'PY' >> gpurun_out/ab_build.log 2>&1
from paper_2305_01867_b200 import _build
_build.build_variant("p21", {"RSI_RAY_PF_L2": 1})
_build.build_variant("p20", {"RSI_RAY_PF_L2": 0})
PY
MODES=boolean,barycentric bash tools/variants.sh "p21 p20 p21 p20" "sphere paper_terrain" > gpurun_out/ab.log 2>&1
