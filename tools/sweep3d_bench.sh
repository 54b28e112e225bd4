#!/bin/bash
# A/B of 3D kernel macros with the default bench (C3 step, device-timed):
# VARIANTS="|-DX=1" [CHUNKS="192 96"] bash tools/sweep3d_bench.sh
mkdir -p gpurun_out
IFS='|' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  touch paper_2511_12235_b200/csrc/mf.cu
  CTSM_NVCC_EXTRA="$v" python -c "from paper_2511_12235_b200 import build as b; b.build()" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for mb in ${CHUNKS:-192}; do
    echo "== [$v] chunk $mb MB: $(CTSM_SYM3D_CHUNK_MB=$mb python bench.py --gpus 1 --steps 6 --warmup 2 --no-cpu --no-e2e --no-clocks ${BENCH_ARGS} | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], r["fwd_ms"], r["bwd_ms"])')"
  done
done
touch paper_2511_12235_b200/csrc/mf.cu
python -c "from paper_2511_12235_b200 import build as b; b.build()" > /dev/null 2>&1
