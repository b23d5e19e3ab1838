cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q -x -k "mle or local_fit or two_stage or theta" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
timeout 600 python scripts/mle_profile.py 2>&1 | tail -1
