#!/bin/bash
# A/B of CSR-emission tuning macros: rebuild with each flag set and run the CSR
# bench. Usage: CFG=c2 VARIANTS="|-DCTSM_CSR3_MINB=5" bash tools/sweep_csr.sh
IFS='|' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  CTSM_NVCC_EXTRA="$v" python -c "from paper_2511_12235_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== [$v] $(python bench.py --mode csr --config ${CFG:-c2} --steps ${STEPS:-1} --warmup 2 --no-clocks 2>&1 | tail -1 | cut -c1-330)"
done
python -c "from paper_2511_12235_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
