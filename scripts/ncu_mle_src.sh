#!/bin/bash
# ncu --set full with source of the MLE kernel on C2 designs (one launch); the report
# comes back for scripts/ncu_lines.py
cd "$GRAFT_REPO_ROOT"
R=${1:-mlex}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mle_kernel -c 1 -o gpurun_out/prof_$R python scripts/mle_profile.py --M 10000 --reps 1 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_$R.ncu-rep > gpurun_out/sum_$R.txt 2>&1
