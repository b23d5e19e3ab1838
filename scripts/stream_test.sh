cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -x -q -k "large_pool or north_star" 2>&1 | tail -3
timeout 1200 python scripts/c5_sweep.py --Nprimes 2000,8000,10000,20000,60000 --ns 50,128 --ps 2,8 --sample 4 --target-ms 300 --out gpurun_out/c5_large_r02a.jsonl > gpurun_out/c5_large.log 2>&1; tail -3 gpurun_out/c5_large.log
