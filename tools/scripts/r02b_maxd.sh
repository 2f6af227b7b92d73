cd $GRAFT_REPO_ROOT
V=paper_2208_01339_b200/variants
timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 10 --libs paper_2208_01339_b200/libnpc.so,$V/libnpc_maxd16.so,paper_2208_01339_b200/libnpc.so,$V/libnpc_maxd16.so 2>&1 | cut -c1-150
