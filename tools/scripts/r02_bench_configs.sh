# r02: one bench line per BASELINE config (+ config 6 DFN) and the reference arm on config 3
for c in 1 2 4 5 6; do
  timeout 900 python bench.py --config $c > gpurun_out/r02_bench_config$c.json 2> gpurun_out/r02_bench_config$c.err; echo "config $c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02_bench_reference_config3.json 2> gpurun_out/r02_bench_reference.err; echo "reference rc=$?"
timeout 900 python bench.py --distributed --steps 2 --warmup 3 > gpurun_out/r02_bench_config3_distributed1.json 2> gpurun_out/r02_bench_dist.err; echo "distributed rc=$?"
