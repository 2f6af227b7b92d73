# r02d: warm-L2 ncu capture of the 128-bit stencil kernel on config 2 (after the plain run)
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/profile_step.py --config 2 --k 30 --iters 2 --applies 2 > gpurun_out/p2v_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_stencil_step_v2 -s 40 -c 1 -o gpurun_out/r02_stencil_step_v2_128_warm python tools/profile_step.py --config 2 --k 30 --iters 2 --applies 2 > gpurun_out/p2v_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/r02_stencil_step_v2_128_warm.ncu-rep --page raw --csv > gpurun_out/r02_ncu_full_stencil_step_v2_128_warm.csv
