#!/bin/bash
# NN phase split for several profiling builds (LIBS), C2 and C4 first chunk
cd "$GRAFT_REPO_ROOT"
for lib in $LIBS; do
  for c in "C2 10000" "C4 65536"; do
   set -- $c
   python scripts/nn_phases.py --config $1 --M $2 --lib $lib
  done
done
