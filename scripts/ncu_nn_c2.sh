cd "$GRAFT_REPO_ROOT"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nn_pool -c 1 -o gpurun_out/prof_nn_c2x python scripts/profile_run.py --M 10000 --form incremental > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_nn_c2x.ncu-rep > gpurun_out/sum_nn_c2x.txt 2>&1
python scripts/ncu_sass_stalls.py gpurun_out/prof_nn_c2x.ncu-rep 60 > gpurun_out/sass_nn_c2x.txt 2>&1
