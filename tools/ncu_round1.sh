set -e
python tools/profile_step.py --config 2 --k 30 --iters 1 --applies 1 > gpurun_out/p2plain.log 2>&1
python tools/profile_step.py --config 5 --k 10 --iters 1 --applies 1 > gpurun_out/p5plain.log 2>&1
python tools/profile_step.py --config 1 --k 10 --iters 1 --applies 1 > gpurun_out/p1plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stencil_step -s 20 -c 1 -o gpurun_out/stencil_full python tools/profile_step.py --config 2 --k 30 --iters 1 --applies 1 > gpurun_out/p2ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_schur_tpass|k_schur_bpass" -s 6 -c 3 -o gpurun_out/schur_full python tools/profile_step.py --config 5 --k 10 --iters 1 --applies 1 > gpurun_out/p5ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_csr_poly_cluster -c 1 -o gpurun_out/cluster_full python tools/profile_step.py --config 1 --k 10 --iters 1 --applies 1 > gpurun_out/p1ncu.log 2>&1
