python -m pytest tests/test_gpu_csr_coded.py tests/test_gpu_parity.py tests/test_gpu_multirank_local.py tests/test_gpu_cluster.py tests/test_gpu_lowrank.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -2
python tools/ab_variants.py --config 3 --k 50 --reps 10 --envs "|NPC_CSR_PLAIN=1|"
