mkdir -p gpurun_out
python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 > gpurun_out/p3plain.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_csr_step -s 60 -c 1 -o gpurun_out/csr_coded_full \
    python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 > gpurun_out/p3ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/csr_coded_full.ncu-rep --page raw --csv > gpurun_out/csr_coded_full_raw.csv
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
