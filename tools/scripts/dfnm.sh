set -x
python -m pytest tests/test_gpu_dfn.py -q -x 2>&1 | tail -3
NPC_DFN_M=1 python -m pytest tests/test_gpu_dfn.py tests/test_gpu_multirank_local.py -q -x -k "dfn" 2>&1 | tail -3
python tools/ab_variants.py --config 6 --k 30 --reps 20 --envs "|NPC_DFN_M=1|" 
