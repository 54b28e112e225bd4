#!/bin/bash
# A/B of 3D kernel tuning macros on the GPU box: rebuild mf.cu with each flag
# set and time the C3 orbit shard (tools/prof3d.py).
# Usage: VARIANTS="|-DCTSM_KZCS=4" bash tools/sweep3d.sh
mkdir -p gpurun_out
IFS='|' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  touch paper_2511_12235_b200/csrc/mf.cu
  CTSM_NVCC_EXTRA="$v" python -c "from paper_2511_12235_b200 import build as b; b.build()" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== [$v] $(python tools/prof3d.py ${CFG:-c3} ${NANG:-64} 2>&1 | tail -1)"
done
touch paper_2511_12235_b200/csrc/mf.cu
python -c "from paper_2511_12235_b200 import build as b; b.build()" > /dev/null 2>&1
