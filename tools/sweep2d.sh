#!/bin/bash
# A/B of 2D kernel tuning macros: rebuild with each flag set and run the C1 bench
# (device-timed value only). Usage: VARIANTS="|-DCTSM_D8F_MINB=5" bash tools/sweep2d.sh
mkdir -p gpurun_out
export CTSM_BENCH_NO_CPU=1
IFS='|' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  CTSM_NVCC_EXTRA="$v" python -c "from paper_2511_12235_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for dt in ${DTYPES:-f64}; do
    echo "== [$v] $dt $(python bench.py --config ${CFG:-c1} --steps 20 --warmup 3 --no-e2e --no-clocks --dtype $dt 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], "fwd", round(r["fwd_ms"],3), "bwd", round(r["bwd_ms"],3))')"
  done
done
python -c "from paper_2511_12235_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
