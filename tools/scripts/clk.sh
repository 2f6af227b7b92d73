for i in 1 2 3; do python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python tools/jsum.py; done
for i in 1 2; do python bench.py --config 4 --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python tools/jsum.py; done
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python tools/jsum.py
