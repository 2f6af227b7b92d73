cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_stencil_grid.py -q -x -p no:cacheprovider > gpurun_out/r02c_grid_tests.log 2>&1; echo "grid tests rc=$?"; tail -15 gpurun_out/r02c_grid_tests.log
timeout 300 python tools/kernel_times.py --config 2 --k 30 --reps 20 > gpurun_out/r02c_kt_grid.txt 2>&1; grep -v arn gpurun_out/r02c_kt_grid.txt | head -5
NPC_NO_GRID_POLY=1 timeout 300 python tools/kernel_times.py --config 2 --k 30 --reps 20 > gpurun_out/r02c_kt_deg.txt 2>&1; grep -v arn gpurun_out/r02c_kt_deg.txt | head -5
timeout 600 python tools/bench_all.py --configs 2 > gpurun_out/r02c_ba2_grid.jsonl 2>/dev/null; echo ba=$?; cut -c1-600 gpurun_out/r02c_ba2_grid.jsonl
NPC_NO_GRID_POLY=1 timeout 600 python tools/bench_all.py --configs 2 > gpurun_out/r02c_ba2_deg.jsonl 2>/dev/null; cut -c1-600 gpurun_out/r02c_ba2_deg.jsonl
