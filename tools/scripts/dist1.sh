# single-GPU vs 1-rank distributed (NCCL) path, same workloads
mkdir -p gpurun_out
for c in "3" "4" "5 --k 50" "2" "6"; do
  for d in "" "--distributed"; do
    echo "== config $c $d"
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e $d 2>/dev/null | python -c "import sys,json; l=json.loads(sys.stdin.readline()); print(json.dumps({k: l[k] for k in ('value','ms_per_step','parallelism')} | {'iters': l['pcg']['iters'], 'apps': l['pcg']['op_applications'], 'frac': l['roofline']['frac']}))"
  done
done 2>&1 | tee gpurun_out/dist1.log
