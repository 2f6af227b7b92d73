cd $GRAFT_REPO_ROOT
V=paper_2208_01339_b200/variants
for lag in 351 450 550 800; do
  NPC_CSR_WAVE=1 NPC_WAVE_LAG=$lag timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_csr_pat_wave -s 5 -c 3 --csv python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 2>/dev/null | grep -E "dram__bytes|duration" | awk -F'","' -v L=$lag '{print "lag", L, $(NF-2), $NF}'
done
AB_INTERVAL=17.6:144820 timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 10 \
  --libs paper_2208_01339_b200/libnpc.so,$V/libnpc_sleep100.so,$V/libnpc_nowait.so --envs "NPC_CSR_WAVE=1|NPC_CSR_WAVE=1,NPC_WAVE_LAG=450|NPC_CSR_WAVE=1,NPC_WAVE_LAG=550" 2>&1 | cut -c1-160
