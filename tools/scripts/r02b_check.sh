cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_csr_pattern.py tests/test_gpu_csr_coded.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 600 python tools/ab_variants.py --config 3 --k 50 --reps 10 --envs "|NPC_CSR_NORING=1|" 2>&1 | cut -c1-150
