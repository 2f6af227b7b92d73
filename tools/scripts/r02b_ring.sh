# r02b: the ring kernel -- parity tests of every CSR form, A/B against k_csr_pat_stage on config 3
# (p_50, 10 applications), then an ncu source-level capture of the ring kernel.
set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_csr_pattern.py tests/test_gpu_csr_coded.py -x -q > gpurun_out/r02b_ring_tests.txt 2>&1
tail -30 gpurun_out/r02b_ring_tests.txt
timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 10 \
  --envs "|NPC_CSR_NORING=1|NPC_RING_NS=2|NPC_RING_NS=3|NPC_CSR_NOFILL=1|NPC_CSR_NORING=1,NPC_CSR_NOFILL=1|" \
  > gpurun_out/r02b_ring_ab.txt 2>&1
cat gpurun_out/r02b_ring_ab.txt
timeout 300 python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 > gpurun_out/p3plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_pat_ring -s 30 -c 1 -o gpurun_out/r02b_csr_pat_ring python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 > gpurun_out/p3ncu.log 2>&1
ncu -i gpurun_out/r02b_csr_pat_ring.ncu-rep --page source --csv --print-source sass > gpurun_out/r02b_pat_ring_source_sass.csv 2>&1
ncu -i gpurun_out/r02b_csr_pat_ring.ncu-rep --page raw --csv > gpurun_out/r02b_pat_ring_raw.csv 2>&1
