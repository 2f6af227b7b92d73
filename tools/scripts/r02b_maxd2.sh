cd $GRAFT_REPO_ROOT
V=paper_2208_01339_b200/variants
L=paper_2208_01339_b200/libnpc.so
timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 30 --libs $L,$V/libnpc_maxd16.so,$L,$V/libnpc_maxd16.so,$L,$V/libnpc_maxd16.so 2>&1 | cut -c1-150
