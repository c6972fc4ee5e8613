#!/bin/bash
# scratch A/B driver (GPU box)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python - <<'PY' >> gpurun_out/ab_build.log 2>&1
from paper_2305_01867_b200 import _build
_build.build_variant("pf", {"RSI_RAY_PREFETCH": 1})
_build.build_variant("nopf", {"RSI_RAY_PREFETCH": 0})
PY
bash tools/variants.sh "pf nopf pf nopf" "sphere paper_terrain" > gpurun_out/ab.log 2>&1
