cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_csr_pattern.py tests/test_gpu_csr_coded.py -q -x 2>&1 | tail -2
V=paper_2208_01339_b200/variants
L=paper_2208_01339_b200/libnpc.so
timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 10 --libs $L,$V/libnpc_noone.so,$L,$V/libnpc_noone.so 2>&1 | cut -c1-150
timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 300 --libs $L,$V/libnpc_noone.so 2>&1 | cut -c1-150
