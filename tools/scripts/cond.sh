NPC_GRAPH_COND=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dfn.py tests/test_gpu_lowrank.py tests/test_gpu_temporal.py -q -x -p no:cacheprovider 2>&1 | tail -2
for c in 2 6 4; do
  python tools/phase_times.py --config $c --reps 5 2>/dev/null | tail -1
  NPC_GRAPH_COND=1 python tools/phase_times.py --config $c --reps 5 2>/dev/null | tail -1
done
python tools/phase_times.py --config 3 --reps 1 2>/dev/null | tail -1
NPC_GRAPH_COND=1 python tools/phase_times.py --config 3 --reps 1 2>/dev/null | tail -1
