set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_csr_pattern.py -q -x > gpurun_out/r02b_wave_tests.txt 2>&1
tail -3 gpurun_out/r02b_wave_tests.txt
V=paper_2208_01339_b200/variants
AB_INTERVAL=17.6:144820 timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 10 \
  --libs paper_2208_01339_b200/libnpc.so,$V/libnpc_nohint.so,$V/libnpc_nowait.so --envs "|NPC_NO_STEP2=1|NPC_WAVE_LAG=400" > gpurun_out/r02b_wave_ab2.txt 2>&1
cat gpurun_out/r02b_wave_ab2.txt
timeout 300 python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 > gpurun_out/p3plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_csr_pat -c 60 --csv --log-file gpurun_out/r02b_wave_ncu.csv python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 > gpurun_out/p3ncu.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r02b_wave_ncu.csv')) if len(r)>10]
h=rows[0]; i=h.index('Kernel Name'); m=h.index('Metric Name'); v=h.index('Metric Value'); u=h.index('Metric Unit'); ID=h.index('ID')
cur=None
for r in rows[1:]:
    if r[ID]!=cur: cur=r[ID]; print(); print(r[ID], r[i][:60], end=' ')
    print(r[m].split('.')[0][:18], r[v], r[u], end='; ')
print()
PY
