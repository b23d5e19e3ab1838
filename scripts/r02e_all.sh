#!/bin/bash
# round-2 evidence after the NN changes: GPU suite, then the round profile (bench line,
# launch list, ncu captures of every hot kernel)
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gputest_${1:-r02e}.log 2>&1; tail -2 gpurun_out/gputest_${1:-r02e}.log
bash scripts/round_profile.sh ${1:-r02e}
