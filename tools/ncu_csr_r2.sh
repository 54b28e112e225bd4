#!/bin/bash
# K1/K2 launch lists (C2 on 8 angles, C0 in full) and one full capture of the
# 3D emission kernel. Usage: TAG=r2c bash tools/ncu_csr_r2.sh
TAG=${TAG:-r2c}
mkdir -p gpurun_out
python tools/prof_csr.py c2 8 > gpurun_out/${TAG}_prof_csr_c2.log 2>&1 || exit 1
python tools/prof_csr.py c0 360 > gpurun_out/${TAG}_prof_csr_c0.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_csr_c2_launches.csv python tools/prof_csr.py c2 8 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_csr_c0_launches.csv python tools/prof_csr.py c0 360 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:emit3d -s 2 -c 1 -f -o gpurun_out/${TAG}_emit3d python tools/prof_csr.py c2 8 > /dev/null 2>&1
ls -la gpurun_out | tail -8
