cd $GRAFT_REPO_ROOT
V=paper_2208_01339_b200/variants
timeout 600 python tools/ab_variants.py --config 2 --k 30 --reps 50 --libs paper_2208_01339_b200/libnpc.so,$V/libnpc_gu2.so,$V/libnpc_gu4.so,$V/libnpc_gu2m3.so,$V/libnpc_gu2m2.so --envs '|NPC_NO_GRID_POLY=1' > gpurun_out/r02c_grid_ab3.txt 2>&1; echo rc=$?; cut -c1-150 gpurun_out/r02c_grid_ab3.txt
