# r02d: evidence at HEAD with the 128-bit stencil kernels as the default: full GPU suite, smoke,
# config 2 bench line, all-config table.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02d_gpu_tests_head.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02d_gpu_tests_head.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02d_smoke.log
timeout 600 python bench.py --config 2 > gpurun_out/r02_bench_config2.json 2> gpurun_out/r02_bench_config2.err; echo "config 2 rc=$?"
timeout 1500 python tools/bench_all.py --configs 1,2 --md gpurun_out/r02_configs_12.md > gpurun_out/r02_bench_all_configs12.jsonl 2> gpurun_out/bench_all.err; echo "bench_all rc=$?"
cat gpurun_out/r02_configs_12.md
