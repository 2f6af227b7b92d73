mkdir -p gpurun_out
for c in 1 2 4 5 6; do
  python bench.py --config $c > gpurun_out/bench_config$c.json 2> gpurun_out/bench_config$c.err; echo "config $c rc=$?"
done
