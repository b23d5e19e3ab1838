#!/bin/bash
# Round evidence (one GPU): the bench line, the launch list of the bench command, and
# ncu --set full captures of every hot kernel at its workload:
#   v2 incremental (C2, C4 first chunk), NN (C2, C4 first chunk), explicit DMMA (C2),
#   MLE (C2 designs), a3 at Fig 4 scale (N' = 60,000, n = 512), HBM-streaming
#   incremental (C5 8-d, N' = 20,000, n = 50).
# usage: bash scripts/round_profile.sh rNN
R=${1:-r02}
cd "$GRAFT_REPO_ROOT"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$R.log 2>&1; tail -1 gpurun_out/bench_$R.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --compare "" > /dev/null 2>&1
NCU="timeout 900 ncu --set full --clock-control none --import-source on -c 1"
$NCU -k regex:alc_incremental_v2 -o gpurun_out/prof_v2_$R python scripts/profile_run.py --M 10000 --form incremental > /dev/null 2>&1
$NCU -k regex:nn_pool -o gpurun_out/prof_nn_$R python scripts/profile_run.py --M 10000 --form incremental > /dev/null 2>&1
$NCU -k regex:alc_incremental_v2 -o gpurun_out/prof_v2_c4_$R python scripts/profile_run.py --config C4 --M 65536 --form incremental > /dev/null 2>&1
$NCU -k regex:nn_pool -o gpurun_out/prof_nn_c4_$R python scripts/profile_run.py --config C4 --M 65536 --form incremental > /dev/null 2>&1
$NCU -k regex:alc_explicit_dmma -o gpurun_out/prof_expl_$R python scripts/profile_run.py --M 10000 --form explicit > /dev/null 2>&1
$NCU -k regex:mle_kernel -o gpurun_out/prof_mle_$R python scripts/mle_profile.py --M 10000 --reps 1 > /dev/null 2>&1
$NCU -k regex:alc_scores_gemm -o gpurun_out/prof_f4_$R python scripts/fig4_sweep.py --nmin 512 --nmax 512 --reps 1 --check "" > /dev/null 2>&1
$NCU -k regex:alc_incremental_stream -o gpurun_out/prof_stream_$R python scripts/profile_run.py --config C5_8d --M 512 --Nprime 20000 --n 50 --form incremental > /dev/null 2>&1
# summaries on the box (the reports together exceed gpurun's 64 MiB copy-back); keep the
# v2 and NN reports
for f in gpurun_out/prof_*_$R.ncu-rep; do
  b=$(basename $f .ncu-rep)
  python scripts/ncu_summary.py $f > gpurun_out/sum_${b#prof_}.txt 2>&1
done
python scripts/traffic_json.py $R C2:incremental:gpurun_out/prof_v2_$R.ncu-rep C2:nn:gpurun_out/prof_nn_$R.ncu-rep \
  C4:incremental:gpurun_out/prof_v2_c4_$R.ncu-rep C4:nn:gpurun_out/prof_nn_c4_$R.ncu-rep \
  C2:explicit:gpurun_out/prof_expl_$R.ncu-rep C2:mle:gpurun_out/prof_mle_$R.ncu-rep \
  F4:scores_gemm:gpurun_out/prof_f4_$R.ncu-rep C5_20000:stream:gpurun_out/prof_stream_$R.ncu-rep > gpurun_out/traffic_$R.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_$R.json
rm -f gpurun_out/prof_nn_c4_$R.ncu-rep gpurun_out/prof_v2_c4_$R.ncu-rep gpurun_out/prof_expl_$R.ncu-rep \
  gpurun_out/prof_mle_$R.ncu-rep gpurun_out/prof_f4_$R.ncu-rep gpurun_out/prof_stream_$R.ncu-rep
ls gpurun_out
