# single-GPU path vs the multi-rank path on a 1-rank NCCL communicator, bench workloads
for c in "3" "4" "5" "5 --k 50" "2" "6" "1"; do
  for d in "" "--distributed"; do
    echo "== config $c $d"
    python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e $d 2>/dev/null | python tools/jsum.py
  done
done
