#!/bin/bash
# compute-sanitizer over the round-2 kernels (small calls via the GPU tests)
cd "$GRAFT_REPO_ROOT"
CS="timeout 1200 compute-sanitizer"
O=gpurun_out/sanitizers_r02.txt
echo "# r02: v2 incremental (256 x 4, TMEM tier, flag publication), HBM-streaming incremental, MLE (128-thread, split buffers), NN (shared-memory selection)" > $O
echo "## memcheck: north_star, large pools (streaming), alc_batch C1 incremental, MLE, NN bit-exact" >> $O
$CS --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_mle.py -q -x -k "north_star or stream_large_pool or (alc_batch_vs_oracle and incremental and C1) or nn_pool_bit_exact or mle_vs_oracle or exhausted" 2>&1 | tail -3 >> $O
echo "## racecheck: streaming kernel (N'=9000) and MLE" >> $O
$CS --tool racecheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_mle.py -q -x -k "stream_large_pool and 9000 or (mle_vs_oracle and 20)" 2>&1 | tail -3 >> $O
echo "## racecheck: NN (shared-memory selection)" >> $O
$CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "nn_pool_bit_exact and C2" 2>&1 | tail -3 >> $O
echo "## synccheck: streaming kernel, MLE, NN" >> $O
$CS --tool synccheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_mle.py -q -x -k "stream_large_pool and 9000 or (mle_vs_oracle and 20) or (nn_pool_bit_exact and C2)" 2>&1 | tail -3 >> $O
echo "## racecheck: v2 incremental (C1 shape, 512 x 1) " >> $O
$CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "alc_batch_vs_oracle and incremental and C1" 2>&1 | tail -3 >> $O
cat $O
