#!/bin/bash
# ncu --set full of the incremental kernel at C2 (10^4 locations): default and LAGP_V2_CPT=4
# usage: bash scripts/ncu_v2.sh TAG
cd "$GRAFT_REPO_ROOT"
T=${1:-x}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:alc_incremental_v2 -c 1 \
  -o gpurun_out/prof_v2_$T python scripts/profile_run.py --M 10000 --form incremental > gpurun_out/ncu_v2_$T.log 2>&1
tail -1 gpurun_out/ncu_v2_$T.log
LAGP_V2_CPT=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:alc_incremental_v2 -c 1 \
  -o gpurun_out/prof_v2c4_$T python scripts/profile_run.py --M 10000 --form incremental > gpurun_out/ncu_v2c4_$T.log 2>&1
tail -1 gpurun_out/ncu_v2c4_$T.log
