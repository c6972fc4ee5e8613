#!/bin/bash
# scratch A/B driver (GPU box): leaf-phase outcome by selects
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python - <<'PY' >> gpurun_out/ab_build.log 2>&1
from paper_2305_01867_b200 import _build
_build.build_variant("ls1", {"RSI_LEAF_SEL": 1})
_build.build_variant("ls0", {"RSI_LEAF_SEL": 0})
PY
bash tools/variants.sh "ls1 ls0 ls1 ls0" "sphere paper_terrain" > gpurun_out/ab.log 2>&1
