# r02d: the fused-allreduce PCG form (tests + 1-rank NCCL A/B), config 2 line with the grid
# kernel at HEAD, all-config table at HEAD.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multirank_local.py -m gpu -q -p no:cacheprovider > gpurun_out/r02d_multirank_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r02d_multirank_tests.log
for c in 3 5; do
  timeout 600 python bench.py --config $c --distributed --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02d_dist_side_c$c.json 2> gpurun_out/r02d_dist_side_c$c.err; echo "side c$c rc=$?"
  NPC_PCG_FUSED_ALLREDUCE=1 timeout 600 python bench.py --config $c --distributed --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02d_dist_fused_c$c.json 2> gpurun_out/r02d_dist_fused_c$c.err; echo "fused c$c rc=$?"
done
python - <<'PY'
import json
for c in (3, 5):
    for m in ("side", "fused"):
        try:
            d = json.load(open(f"gpurun_out/r02d_dist_{m}_c{c}.json"))
            print(c, m, d["ms_per_step"], d["pcg"]["iters"], d["pcg"]["op_applications"], d["pcg"]["reductions"])
        except Exception as e:
            print(c, m, "failed", e)
PY
timeout 600 python bench.py --config 2 > gpurun_out/r02_bench_config2.json 2> gpurun_out/r02_bench_config2.err; echo "config 2 rc=$?"
timeout 1500 python tools/bench_all.py --configs 1,2,3,4,5,6 --md gpurun_out/r02_configs.md > gpurun_out/r02_bench_all_configs1to6.jsonl 2> gpurun_out/bench_all.err; echo "bench_all rc=$?"
cat gpurun_out/r02_configs.md
