cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_csr_pattern.py tests/test_gpu_csr_coded.py tests/test_gpu_multirank_local.py tests/test_gpu_cluster.py -q -x 2>&1 | tail -2
NPC_CREATE_TIMES=1 timeout 600 python tools/create_times.py --configs 3 2>&1 | tail -8
