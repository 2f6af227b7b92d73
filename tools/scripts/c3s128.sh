for t in "" "--no-kernel-timing"; do
for d in "" "--distributed"; do
  echo "== $t $d"
  python bench.py --config 3 --side 128 --steps 2 --warmup 3 --no-cpu --no-e2e $t $d 2>/dev/null | python tools/jsum.py
done; done
