#!/bin/bash
# compute-sanitizer over the NN kernel after the multi-axis cell grid, the value-bin
# selection and the work counters (small calls via the GPU tests)
cd "$GRAFT_REPO_ROOT"
CS="timeout 1500 compute-sanitizer"
O=gpurun_out/sanitizers_r02f.txt
echo "# r02f: NN multi-axis cell lists, one-pass value-bin selection, work counters; MLE (interleaved DMMA chains)" > $O
echo "## memcheck: NN multi-axis edge cases (sorted + selected), C2 NN bit-exact, counters, MLE" >> $O
$CS --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_mle.py -q -x -k "(multi_cells and 1000) or (selected and 1000-6) or (nn_pool_bit_exact and C2) or counters or (mle_vs_oracle and 20)" 2>&1 | tail -3 >> $O
echo "## racecheck: NN (multi-axis lists, C2 bit-exact; selected pools)" >> $O
$CS --tool racecheck python -m pytest -q -x "tests/test_gpu_parity.py::test_nn_pool_bit_exact[C2-48-None-1000]" "tests/test_gpu_parity.py::test_nn_pool_selected_bit_exact[1000-6-1]" "tests/test_gpu_parity.py::test_nn_pool_multi_cells_bit_exact[1000-2]" 2>&1 | tail -3 >> $O
echo "## synccheck: NN, MLE" >> $O
$CS --tool synccheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_mle.py -q -x -k "(nn_pool_bit_exact and C2) or (mle_vs_oracle and 20)" 2>&1 | tail -3 >> $O
echo "## racecheck: MLE" >> $O
$CS --tool racecheck python -m pytest tests/test_gpu_mle.py -q -x -k "mle_vs_oracle and 20" 2>&1 | tail -3 >> $O
cat $O
