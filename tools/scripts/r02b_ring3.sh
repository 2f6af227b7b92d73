set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_csr_pattern.py tests/test_gpu_csr_coded.py -q > gpurun_out/r02b_ring_tests.txt 2>&1
tail -5 gpurun_out/r02b_ring_tests.txt
V=paper_2208_01339_b200/variants
timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps 10 \
  --libs paper_2208_01339_b200/libnpc.so,$V/libnpc_prev.so,$V/libnpc_w1k.so,$V/libnpc_w200k.so,paper_2208_01339_b200/libnpc.so > gpurun_out/r02b_ring_ab3.txt 2>&1
cat gpurun_out/r02b_ring_ab3.txt
timeout 900 python bench.py --no-cpu > gpurun_out/r02b_bench3.json 2> gpurun_out/r02b_bench3.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02b_bench3.json')); r=d['roofline']
print(d['ms_per_step'], d['pcg']['iters'], r['frac'], r['launch_ms'], r['isolated_achieved'], d['clocks'], {k:(v['ms']/v['launches']) for k,v in r['step_breakdown'].items()})"
