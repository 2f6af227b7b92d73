set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_csr_pattern.py tests/test_gpu_csr_coded.py -q -x > gpurun_out/r02b_wave_tests.txt 2>&1
tail -25 gpurun_out/r02b_wave_tests.txt
timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 10 \
  --envs "|NPC_NO_STEP2=1|NPC_WAVE_LAG=150|NPC_WAVE_LAG=600|NPC_WAVE_LAG=1200|" > gpurun_out/r02b_wave_ab.txt 2>&1
cat gpurun_out/r02b_wave_ab.txt
timeout 600 python tools/ab_variants.py --config 3 --k 50 --reps 10 --libs paper_2208_01339_b200/variants/libnpc_nohint.so >> gpurun_out/r02b_wave_ab.txt 2>&1
tail -1 gpurun_out/r02b_wave_ab.txt
