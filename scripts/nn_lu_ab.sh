#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for cr in ${CRS:-128}; do
  for c in "C2 10000" "C4 65536"; do
   set -- $c
   LAGP_NN_CR=$cr python scripts/nn_phases.py --config $1 --M $2 --lib ${LIB:-liblagp_b200_prof.so}
  done
done
