cd $GRAFT_REPO_ROOT
V=paper_2208_01339_b200/variants
timeout 600 python tools/ab_variants.py --config 2 --k 30 --reps 50 --libs paper_2208_01339_b200/libnpc.so,$V/libnpc_gminb5.so,$V/libnpc_gminb3.so --envs '|NPC_NO_GRID_POLY=1|NPC_GRID_ZC=8|NPC_GRID_ZC=4' > gpurun_out/r02c_grid_ab2.txt 2>&1; echo rc=$?; cut -c1-150 gpurun_out/r02c_grid_ab2.txt
timeout 600 python -m pytest tests/test_gpu_stencil_grid.py -q -x -p no:cacheprovider > gpurun_out/r02c_grid_tests2.log 2>&1; echo "grid tests rc=$?"; tail -3 gpurun_out/r02c_grid_tests2.log
