cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_csr_pattern.py -q -x 2>&1 | tail -3
AB_INTERVAL=17.6:144820 timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 10 \
  --envs "|NPC_CSR_WAVE=1|NPC_CSR_WAVE=1,NPC_WAVE_PERSIST=1|NPC_CSR_WAVE=1,NPC_WAVE_PERSIST=1,NPC_WAVE_LAG=450|NPC_CSR_WAVE=1,NPC_WAVE_PERSIST=1,NPC_WAVE_LAG=700" 2>&1 | cut -c1-150
for ev in "NPC_CSR_WAVE=1 NPC_WAVE_PERSIST=1" ""; do
  env $ev timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/instep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/instep.json')); r=d['roofline']
print('$ev' or 'default', d['ms_per_step'], d['pcg']['iters'], r['launch_ms'], d['clocks']['sm_mhz'], d['clocks']['power_w_median'], {k:round(v['ms']/v['launches'],4) for k,v in r['step_breakdown'].items()})"
done
