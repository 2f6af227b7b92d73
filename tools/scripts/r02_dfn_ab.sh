# r02 DFN A/B: L2 prefetch of A_f^-1 off, evict-last first pass (time + DRAM bytes per k_dfn_dense launch)
L=paper_2208_01339_b200/libnpc.so,paper_2208_01339_b200/variants/libnpc_nopfai.so,paper_2208_01339_b200/variants/libnpc_evl.so,paper_2208_01339_b200/variants/libnpc_evlnopf.so
timeout 900 python tools/ab_variants.py --config 6 --k 30 --reps 10 --libs $L > gpurun_out/r02_dfn_ab.log 2>&1
for v in libnpc.so variants/libnpc_nopfai.so variants/libnpc_evl.so variants/libnpc_evlnopf.so; do
  NPC_LIB_PATH=paper_2208_01339_b200/$v timeout 300 python tools/profile_step.py --config 6 --k 30 --iters 1 --applies 1 > gpurun_out/p6plain.log 2>&1 && \
  NPC_LIB_PATH=paper_2208_01339_b200/$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_dfn_dense -s 20 -c 3 --csv python tools/profile_step.py --config 6 --k 30 --iters 1 --applies 1 > gpurun_out/r02_dfn_ncu_$(basename $v .so).csv 2>&1
done
