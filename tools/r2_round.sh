#!/bin/bash
# One GPU round trip (round 2): parity suite, the default bench line (C3), the
# reference arm with the driver's flags, and the other workloads' lines.
# Usage (repo root, via gpurun): TAG=r2b bash tools/r2_round.sh
mkdir -p gpurun_out
TAG=${TAG:-r2x}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; tail -1 gpurun_out/smoke_${TAG}.log
if [ -z "$NO_TESTS" ]; then
CTSM_PARITY_REPORT=gpurun_out/parity_${TAG}.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; tail -5 gpurun_out/pytest_${TAG}.log
fi
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_c3_f32_${TAG}.json 2> gpurun_out/bench_c3_f32_${TAG}.err; tail -1 gpurun_out/bench_c3_f32_${TAG}.json
if [ -z "$NO_REF" ]; then
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_reference_c3_${TAG}.json 2>&1; tail -1 gpurun_out/bench_reference_c3_${TAG}.json
fi
if [ -z "$NO_OTHERS" ]; then
python bench.py --config c1 > gpurun_out/bench_c1_f64_${TAG}.json 2>&1; tail -1 gpurun_out/bench_c1_f64_${TAG}.json
python bench.py --config c1 --dtype f32 --no-cpu > gpurun_out/bench_c1_f32_${TAG}.json 2>&1; tail -1 gpurun_out/bench_c1_f32_${TAG}.json
python bench.py --config c4 --mode sirt --steps 2 --warmup 2 > gpurun_out/bench_sirt_c4_f32_${TAG}.json 2>&1; tail -1 gpurun_out/bench_sirt_c4_f32_${TAG}.json
python bench.py --config c0 --mode csr > gpurun_out/bench_csr_c0_${TAG}.json 2>&1; tail -1 gpurun_out/bench_csr_c0_${TAG}.json
python bench.py --config c2 --mode csr --steps 2 --warmup 1 > gpurun_out/bench_csr_c2_${TAG}.json 2>&1; tail -1 gpurun_out/bench_csr_c2_${TAG}.json
fi
ls gpurun_out
