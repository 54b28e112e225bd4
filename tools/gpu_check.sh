#!/bin/bash
# One GPU round trip: parity tests + benches (run via gpurun from the repo root).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
if [ -n "$PYTEST_K" ]; then KARGS=(-k "$PYTEST_K"); else KARGS=(); fi
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -p no:cacheprovider "${KARGS[@]}" > gpurun_out/pytest.log 2>&1; tail -25 gpurun_out/pytest.log
for spec in ${BENCHES:-"c1:f64"}; do
  cfg=${spec%%:*}; dt=${spec##*:}
  timeout 900 python bench.py --config $cfg --dtype $dt --steps ${STEPS:-5} --warmup ${WARMUP:-3} > gpurun_out/bench_${cfg}_${dt}.log 2>&1
  tail -1 gpurun_out/bench_${cfg}_${dt}.log
done
