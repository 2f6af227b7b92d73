set -e
mkdir -p gpurun_out
python tools/profile_step.py --config 6 --k 30 --iters 1 --applies 1 > gpurun_out/p6plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_dfn_dense|k_dfn_out" -s 4 -c 2 -o gpurun_out/dfn_full python tools/profile_step.py --config 6 --k 30 --iters 1 --applies 1 > gpurun_out/p6ncu.log 2>&1
ncu -i gpurun_out/dfn_full.ncu-rep --page raw --csv > gpurun_out/dfn_full_raw.csv
ncu -i gpurun_out/dfn_full.ncu-rep --page source --csv -k regex:k_dfn_dense > gpurun_out/dfn_full_src.csv 2>/dev/null || true
echo ok
