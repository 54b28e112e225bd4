#!/bin/bash
# A/B of CSR SpMV variants (K3) on the C2 matrix: rebuild with each flag set
# and run the CSR bench (assembly + SpMV). Usage: VARIANTS="|-DCTSM_SPMV_V=1" bash tools/sweep_spmv.sh
mkdir -p gpurun_out
IFS='|' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  CTSM_NVCC_EXTRA="$v" python -c "from paper_2511_12235_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== [$v] $(python bench.py --mode csr --config ${CFG:-c2} --steps 1 --warmup 3 --no-clocks 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], "spmv", d["spmv"])')"
done
python -c "from paper_2511_12235_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
