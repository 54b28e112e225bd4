#!/bin/bash
# A/B of runtime knobs (environment) for the 3D kernels: ENVS="A=1|B=2" bash tools/sweep3d_env.sh
IFS='|' read -ra VS <<< "${ENVS}"
for v in "${VS[@]}"; do
  echo "== [$v] $(env $v python tools/prof3d.py ${CFG:-c3} ${NANG:-64} 2>&1 | tail -1)"
done
