cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02b_gpu_tests_head.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02b_gpu_tests_head.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
