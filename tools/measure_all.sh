#!/bin/bash
# One GPU round trip for the committed numbers: bench lines (C1 f64/f32, C3
# f32, C4 SIRT f32), the C1 launch list and ncu --set full captures of the 2D
# and 3D kernels. Usage (from the repo root, via gpurun): TAG=r1q bash tools/measure_all.sh
mkdir -p gpurun_out
TAG=${TAG:-rx}
python bench.py > gpurun_out/bench_c1_f64_${TAG}.log 2>&1; tail -1 gpurun_out/bench_c1_f64_${TAG}.log
python bench.py --dtype f32 > gpurun_out/bench_c1_f32_${TAG}.log 2>&1; tail -1 gpurun_out/bench_c1_f32_${TAG}.log
python bench.py --config c3 --dtype f32 --steps 3 --warmup 3 > gpurun_out/bench_c3_f32_${TAG}.log 2>&1; tail -1 gpurun_out/bench_c3_f32_${TAG}.log
if [ -z "$NO_SIRT" ]; then
python bench.py --config c4 --dtype f32 --mode sirt --steps 2 --warmup 3 > gpurun_out/bench_sirt_c4_f32_${TAG}.log 2>&1; tail -1 gpurun_out/bench_sirt_c4_f32_${TAG}.log
fi
TAG=$TAG bash tools/ncu_2d.sh
TAG=$TAG bash tools/ncu_3d.sh
ls gpurun_out
