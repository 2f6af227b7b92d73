# in-step A/B of the CSR degree kernels on the full config-3 solve (bench, no CPU / e2e legs)
cd $GRAFT_REPO_ROOT
for ev in "" "NPC_CSR_WAVE=1" "NPC_RING_RPT=4" ""; do
  env $ev timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/instep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/instep.json')); r=d['roofline']
print('$ev' or 'default', d['ms_per_step'], d['pcg']['iters'], r['launch_ms'], d['clocks']['sm_mhz'], d['clocks']['power_w_median'], {k:round(v['ms']/v['launches'],4) for k,v in r['step_breakdown'].items()})"
done
