cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_csr_pattern.py tests/test_gpu_csr_coded.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/instep.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/instep.json')); r=d['roofline']
print(d['ms_per_step'], d['pcg']['iters'], r['launch_ms'], d['clocks']['sm_mhz'], {k:round(v['ms']/v['launches'],4) for k,v in r['step_breakdown'].items()})"
