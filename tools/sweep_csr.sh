#!/bin/bash
# A/B of CSR-emission tuning macros: rebuild csr.cu with each flag set and run
# the CSR bench. Usage: CFG=c2 VARIANTS="|-DCTSM_EMIT3_MINB=5" bash tools/sweep_csr.sh
IFS='|' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  touch paper_2511_12235_b200/csrc/csr.cu
  CTSM_NVCC_EXTRA="$v" python -c "from paper_2511_12235_b200 import build as b; b.build()" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== [$v] $(python bench.py --mode csr --config ${CFG:-c2} --steps ${STEPS:-2} --warmup 1 --no-clocks --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-230)"
done
touch paper_2511_12235_b200/csrc/csr.cu
python -c "from paper_2511_12235_b200 import build as b; b.build()" > /dev/null 2>&1
