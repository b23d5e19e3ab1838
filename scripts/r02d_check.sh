cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02d.log 2>&1; tail -1 gpurun_out/bench_r02d.log | cut -c1-400
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gputest_r02d.log 2>&1; tail -3 gpurun_out/gputest_r02d.log
