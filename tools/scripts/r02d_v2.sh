# r02d: k_stencil_step_v2 (two x-points per thread, 128-bit accesses): tests, eager p_30 A/B,
# PCG solve A/B on config 2, the multi-rank stencil cases through it.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stencil_vec2.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02d_v2_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r02d_v2_tests.log
NPC_ST_V2=1 timeout 900 python -m pytest tests/test_gpu_multirank_local.py tests/test_gpu_parity.py -m gpu -q -k "stencil or c2" -p no:cacheprovider > gpurun_out/r02d_v2_multirank.log 2>&1; echo "multirank rc=$?"
tail -3 gpurun_out/r02d_v2_multirank.log
timeout 600 python tools/ab_variants.py --config 2 --k 30 --reps 50 --envs 'NPC_NO_GRID_POLY=1|NPC_NO_GRID_POLY=1,NPC_ST_V2=1|NPC_NO_GRID_POLY=1|NPC_NO_GRID_POLY=1,NPC_ST_V2=1|' > gpurun_out/r02d_v2_ab.txt 2>&1; echo rc=$?; cut -c1-300 gpurun_out/r02d_v2_ab.txt
timeout 600 python tools/scripts/r02d_v2_solve_ab.py > gpurun_out/r02d_v2_solve_ab.txt 2>&1; echo rc=$?; cat gpurun_out/r02d_v2_solve_ab.txt
