# r02: TMA two-degree pass (k_stencil_tma2, opt-in) vs the one-degree TMA kernel and the register kernels
timeout 900 python -m pytest tests/test_gpu_temporal.py tests/test_gpu_stencil_tma.py tests/test_gpu_cluster.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r02_st5.log 2>&1; echo rc=$? >> gpurun_out/r02_st5.log
for side in 128 256; do
  echo "side $side" >> gpurun_out/r02_st5.log
  timeout 600 python tools/ab_variants.py --config 2 --side $side --k 30 --reps 10 --envs "|NPC_ST_TMA2=1|NPC_ST_NOTMA=1,NPC_NO_STEP2=1" >> gpurun_out/r02_st5.log 2>&1
done
