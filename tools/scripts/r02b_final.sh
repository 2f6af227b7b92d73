# r02b round-end evidence at HEAD: GPU tests, smoke, the headline kernel's ncu capture (traffic
# file), the default bench line and its launch list, one bench line per config, the reference
# arm, the distributed 1-rank path and the all-config table.  Each ncu command after the same
# command exited 0 without ncu.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02b_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02b_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02b_smoke.log
timeout 300 python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 > gpurun_out/p3plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_pat_ring -s 30 -c 1 -o gpurun_out/r02_csr_pat_ring python tools/profile_step.py --config 3 --k 50 --iters 1 --applies 1 > gpurun_out/p3ncu.log 2>&1
ncu -i gpurun_out/r02_csr_pat_ring.ncu-rep --page raw --csv > gpurun_out/r02_ncu_full_csr_pat_ring.csv
ncu -i gpurun_out/r02_csr_pat_ring.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_ncu_source_csr_pat_ring.csv 2>&1
MB=$(python -c "
import sys; sys.path.insert(0, '.')
import bench, paper_2208_01339_b200 as npc
w = bench.make_workload(3, None); ctx = npc.npc_context_create(0); op = npc.create_from_workload(ctx, w, 'csr')
print(npc.npc_operator_matrix_bytes(op), w['n'])")
set -- $MB
python tools/traffic_from_ncu.py gpurun_out/r02_ncu_full_csr_pat_ring.csv 3 $(python -c "print($1 + 32 * $2)") $1 50
cp profiles/traffic_config3.json gpurun_out/traffic_config3.json
timeout 900 python bench.py > gpurun_out/r02_bench_config3.json 2> gpurun_out/r02_bench_config3.err; echo "bench rc=$?"
head -c 300 gpurun_out/r02_bench_config3.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r02_launches_bench_config3.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
bash tools/scripts/r02_bench_configs.sh
timeout 1500 python tools/bench_all.py --configs 1,2,3,4,5,6 --md gpurun_out/r02_configs.md > gpurun_out/r02_bench_all_configs1to6.jsonl 2> gpurun_out/bench_all.err; echo "bench_all rc=$?"
cat gpurun_out/r02_configs.md
