set -x
python -m pytest tests/test_gpu_multirank_local.py tests/test_gpu_lowrank.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -4
for c in "5 --k 50" "2" "6" "3 --side 128" "4"; do
  for d in "" "--distributed"; do
    echo "== config $c $d"
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e $d 2>/dev/null | python -c "import sys,json; l=json.loads(sys.stdin.readline()); print(json.dumps({k: l[k] for k in ('value','ms_per_step','parallelism')} | {'iters': l['pcg']['iters'], 'apps': l['pcg']['op_applications'], 'red': l['pcg']['reductions'], 'frac': l['roofline']['frac']}))"
  done
done
