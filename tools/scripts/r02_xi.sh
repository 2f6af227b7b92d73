timeout 1200 python -m pytest tests/test_gpu_xi.py -x -q -m gpu > gpurun_out/r02_xi_tests.log 2>&1; echo rc=$? >> gpurun_out/r02_xi_tests.log
timeout 900 python tools/xi_sweep.py --configs 1,2,4 --reps 3 --md gpurun_out/r02_xi_sweep_124.md --jsonl gpurun_out/r02_xi_sweep_124.jsonl > gpurun_out/r02_xi_124.log 2>&1
timeout 1500 python tools/xi_sweep.py --configs 3 --reps 1 --md gpurun_out/r02_xi_sweep_3.md --jsonl gpurun_out/r02_xi_sweep_3.jsonl > gpurun_out/r02_xi_3.log 2>&1
