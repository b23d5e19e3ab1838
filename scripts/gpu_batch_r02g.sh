cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "deep_design" 2>&1 | tail -2
for q in 4 8 16; do LAGP_NN_Q=$q python scripts/lib_ab.py --flush --reps 5 --libs liblagp_b200.so | sed "s/^/Q=$q /"; done
bash scripts/sanitize_r02f.sh
