cd $GRAFT_REPO_ROOT
V=paper_2208_01339_b200/variants
L=paper_2208_01339_b200/libnpc.so
timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 10 --libs $L,$V/libnpc_t512.so --envs "|NPC_RING_NS=2|NPC_RING_NS=2,NPC_RING_RPT=4" 2>&1 | cut -c1-150
