#!/bin/bash
# A/B of NN sampling parameters (experiment builds liblagp_nn_<S2F>_<TGT>.so) at C2 and C4
cd "$GRAFT_REPO_ROOT"
for lib in "" paper_1310_5182_b200/liblagp_nn_128_125.so paper_1310_5182_b200/liblagp_nn_256_115.so paper_1310_5182_b200/liblagp_nn_128_15.so; do
  L=""; [ -n "$lib" ] && L="--lib $lib"
  echo "== ${lib:-default}"
  python scripts/profile_run.py --M 10000 --form incremental --reps 3 $L | tail -1
  python scripts/profile_run.py --config C4 --M 65536 --form incremental --reps 2 $L | tail -1
  python scripts/profile_run.py --config C3 --M 100000 --form incremental --reps 2 $L | tail -1
done
