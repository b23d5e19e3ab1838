#!/bin/bash
# C5 large pools on the incremental form (HBM-streaming kernel beyond N' = 8192), and
# the A/B of the streaming kernel against the v1 kernel for 1024 < N' <= 8192
cd "$GRAFT_REPO_ROOT"
timeout 2400 python scripts/c5_sweep.py --Nprimes 10000,20000,60000 --ns 50,128 --ps 2,8 --forms incremental --sample 4 --target-ms 300 --out gpurun_out/c5_stream_r02.jsonl > gpurun_out/c5_stream.log 2>&1; tail -2 gpurun_out/c5_stream.log
LAGP_INC_STREAM=1 timeout 1200 python scripts/c5_sweep.py --Nprimes 2000,5000,8000 --ns 50,128 --ps 2,8 --forms incremental --sample 2 --target-ms 300 --out gpurun_out/c5_stream_mid_r02.jsonl > gpurun_out/c5_stream_mid.log 2>&1; tail -2 gpurun_out/c5_stream_mid.log
