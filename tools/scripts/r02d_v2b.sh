# r02d: 128-bit stencil kernels as the default (per-degree and cooperative): tests, p_30 A/B
# (grid vs per-degree, CTAs per SM of the grid kernel, z-chunks), PCG solve A/B on config 2.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_stencil_vec2.py tests/test_gpu_stencil_grid.py tests/test_gpu_stencil_tma.py tests/test_gpu_temporal.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02d_v2b_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02d_v2b_tests.log
V=paper_2208_01339_b200/variants
timeout 900 python tools/ab_variants.py --config 2 --k 30 --reps 50 --libs paper_2208_01339_b200/libnpc.so,$V/libnpc_gv2_6.so,$V/libnpc_gv2_4.so --envs '|NPC_ST_NOV2=1' > gpurun_out/r02d_v2b_ab_grid.txt 2>&1; echo rc=$?; cut -c1-200 gpurun_out/r02d_v2b_ab_grid.txt
timeout 900 python tools/ab_variants.py --config 2 --k 30 --reps 50 --envs 'NPC_NO_GRID_POLY=1|NPC_NO_GRID_POLY=1,NPC_ST_ZC=4|NPC_NO_GRID_POLY=1,NPC_ST_ZC=16|NPC_NO_GRID_POLY=1,NPC_ST_ZC=6|NPC_NO_GRID_POLY=1,NPC_ST_NOV2=1' > gpurun_out/r02d_v2b_ab_step.txt 2>&1; echo rc=$?; cut -c1-200 gpurun_out/r02d_v2b_ab_step.txt
timeout 600 python tools/scripts/r02d_v2_solve_ab.py > gpurun_out/r02d_v2b_solve_ab.txt 2>&1; echo rc=$?; cat gpurun_out/r02d_v2b_solve_ab.txt
