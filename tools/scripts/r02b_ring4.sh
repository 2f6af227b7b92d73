set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_csr_pattern.py tests/test_gpu_csr_coded.py -q > gpurun_out/r02b_ring_tests.txt 2>&1
tail -5 gpurun_out/r02b_ring_tests.txt
timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 10 \
  --envs "|NPC_RING_RPT=4|NPC_RING_NS=2|NPC_RING_NS=2,NPC_RING_RPT=4|" > gpurun_out/r02b_ring_ab4.txt 2>&1
cat gpurun_out/r02b_ring_ab4.txt
(nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 200 > gpurun_out/r02b_clk_long.txt) & SMI=$!
timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 400 --envs "|NPC_RING_RPT=4" > gpurun_out/r02b_ring_ab4_long.txt 2>&1
kill $SMI
cat gpurun_out/r02b_ring_ab4_long.txt
