# r02d: round-end evidence at HEAD: full GPU suite, smoke, default bench line (config 3),
# config 2 line, all-config table, launch list of the config-2 bench command.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02d_gpu_tests_head.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02d_gpu_tests_head.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02d_smoke.log
timeout 900 python bench.py > gpurun_out/r02_bench_config3.json 2> gpurun_out/r02_bench_config3.err; echo "bench rc=$?"
timeout 600 python bench.py --config 2 > gpurun_out/r02_bench_config2.json 2> gpurun_out/r02_bench_config2.err; echo "config 2 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench_config2.csv python bench.py --config 2 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_c2.log 2>&1; echo "launch list rc=$?"
timeout 1500 python tools/bench_all.py --configs 1,2,3,4,5,6 --md gpurun_out/r02_configs.md > gpurun_out/r02_bench_all_configs1to6.jsonl 2> gpurun_out/bench_all.err; echo "bench_all rc=$?"
cat gpurun_out/r02_configs.md
