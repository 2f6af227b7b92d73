# r02d: programmatic dependent launch of k_stencil_step_v2 (opt-in NPC_ST_PDL=1): tests under
# it, eager p_30 A/B and PCG solve A/B on config 2.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NPC_ST_PDL=1 timeout 900 python -m pytest tests/test_gpu_stencil_vec2.py tests/test_gpu_stencil_grid.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02d_pdl_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02d_pdl_tests.log
timeout 900 python tools/ab_variants.py --config 2 --k 30 --reps 50 --envs '|NPC_ST_PDL=1||NPC_ST_PDL=1' > gpurun_out/r02d_pdl_ab.txt 2>&1; echo rc=$?; cut -c1-200 gpurun_out/r02d_pdl_ab.txt
timeout 600 python tools/scripts/r02d_pdl_solve_ab.py > gpurun_out/r02d_pdl_solve_ab.txt 2>&1; echo rc=$?; cat gpurun_out/r02d_pdl_solve_ab.txt
