# r02b diagnostics of the headline pattern kernel: A/B of the earlier-tile L2 mirror reads and
# of the row sums (variants wrong on purpose, fixed interval), then an ncu source-level capture.
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
AB_INTERVAL=17.6:144820 python tools/ab_variants.py --config 3 --k 50 --reps 10 \
  --libs paper_2208_01339_b200/libnpc.so,paper_2208_01339_b200/variants/libnpc_nol2m.so,paper_2208_01339_b200/variants/libnpc_nosum.so,paper_2208_01339_b200/libnpc.so \
  > gpurun_out/r02b_ab_diag.txt 2>&1
cat gpurun_out/r02b_ab_diag.txt
python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 > gpurun_out/p3plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_pat_stage -s 30 -c 1 -o gpurun_out/r02b_csr_pat_stage python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 > gpurun_out/p3ncu.log 2>&1
ncu -i gpurun_out/r02b_csr_pat_stage.ncu-rep --page source --csv --print-source sass > gpurun_out/r02b_pat_stage_source_sass.csv 2>&1
ncu -i gpurun_out/r02b_csr_pat_stage.ncu-rep --page source --csv --print-source cuda > gpurun_out/r02b_pat_stage_source_cuda.csv 2>&1
ls -la gpurun_out
