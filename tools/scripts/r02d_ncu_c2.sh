# r02d: warm-L2 ncu captures of config 2's kernels (128^3 stencil, vectors L2-resident):
# one per-degree k_stencil_step launch deep inside p_30, and the cooperative all-degree kernel.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/profile_step.py --config 2 --k 30 --iters 2 --applies 2 > gpurun_out/p2c_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_stencil_step -s 40 -c 1 -o gpurun_out/r02_stencil_step128_warm python tools/profile_step.py --config 2 --k 30 --iters 2 --applies 2 > gpurun_out/p2c_ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_stencil_poly_grid -s 1 -c 1 -o gpurun_out/r02_stencil_grid128_warm python tools/profile_step.py --config 2 --k 30 --iters 2 --applies 2 > gpurun_out/p2c_ncu2.log 2>&1; echo "ncu2 rc=$?"
for f in r02_stencil_step128_warm r02_stencil_grid128_warm; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/r02_ncu_full_${f#r02_}.csv
done
ls -la gpurun_out/*.ncu-rep
