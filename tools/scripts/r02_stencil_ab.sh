timeout 900 python -m pytest tests/test_gpu_stencil_tma.py tests/test_gpu_temporal.py -x -q -m gpu > gpurun_out/r02_st3.log 2>&1; echo rc=$? >> gpurun_out/r02_st3.log
L=paper_2208_01339_b200/libnpc.so,paper_2208_01339_b200/variants/libnpc_ns5.so,paper_2208_01339_b200/variants/libnpc_ns6.so,paper_2208_01339_b200/variants/libnpc_ty8.so
for side in 200 256; do
  echo "side $side" >> gpurun_out/r02_st3.log
  timeout 600 python tools/ab_variants.py --config 2 --side $side --k 30 --reps 10 --libs $L --envs "|NPC_ST_TZC=32" >> gpurun_out/r02_st3.log 2>&1
done
timeout 300 python tools/ab_variants.py --config 2 --side 256 --k 30 --reps 10 --envs "NPC_ST_NOTMA=1|NPC_STEP2=1" >> gpurun_out/r02_st3.log 2>&1
