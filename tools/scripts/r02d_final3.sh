set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02d_gpu_tests_head.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02d_gpu_tests_head.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02d_smoke.log
timeout 600 python bench.py --config 2 > gpurun_out/r02_bench_config2.json 2> gpurun_out/r02_bench_config2.err; echo "config 2 rc=$?"
timeout 900 python bench.py > gpurun_out/r02_bench_config3.json 2> gpurun_out/r02_bench_config3.err; echo "bench rc=$?"
