# round-end: full GPU tests, smoke, default bench line, reference arm, all-config table
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python tools/bench_all.py --configs 1,2,3,4,5,6 --md gpurun_out/r01_configs.md > gpurun_out/bench_all.jsonl 2> gpurun_out/bench_all.err; echo "bench_all rc=$?"
cat gpurun_out/r01_configs.md
