set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_csr_pattern.py tests/test_gpu_csr_coded.py -q > gpurun_out/r02b_ring_tests.txt 2>&1
tail -15 gpurun_out/r02b_ring_tests.txt
timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 10 \
  --envs "|NPC_CSR_NORING=1|NPC_RING_NS=2|NPC_CSR_NOFILL=1|" > gpurun_out/r02b_ring_ab2.txt 2>&1
cat gpurun_out/r02b_ring_ab2.txt
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02b_gpu_tests.txt 2>&1
tail -15 gpurun_out/r02b_gpu_tests.txt
