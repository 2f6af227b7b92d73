cd $GRAFT_REPO_ROOT
V=paper_2208_01339_b200/variants
L=paper_2208_01339_b200/libnpc.so
timeout 900 python tools/ab_variants.py --config 2 --k 30 --reps 20 --libs $L,$V/libnpc_stu2.so,$V/libnpc_stu4.so,$V/libnpc_stu8.so,$L --envs "|NPC_ST_ZC=4|NPC_ST_ZC=16" 2>&1 | cut -c1-170
