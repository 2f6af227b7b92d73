# r02 evidence: full ncu capture of the headline kernel (config 3 pattern form) and the 256^3
# TMA stencil kernel, and the launch list of the bench command.  Each ncu command runs after the
# same command exited 0 without ncu.
set -e
python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 > gpurun_out/p3plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_csr_pat_stage -s 30 -c 1 -o gpurun_out/r02_csr_pat_stage python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 > gpurun_out/p3ncu.log 2>&1
python tools/profile_step.py --config 2 --side 256 --k 30 --iters 1 --applies 1 > gpurun_out/p2plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stencil_tma -s 30 -c 1 -o gpurun_out/r02_stencil_tma256 python tools/profile_step.py --config 2 --side 256 --k 30 --iters 1 --applies 1 > gpurun_out/p2ncu.log 2>&1
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02_bench_plain.json 2> gpurun_out/r02_bench_plain.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches_bench_config3.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02_bench_ncu.log 2>&1
