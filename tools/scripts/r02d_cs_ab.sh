# r02d: k_cg_update with streaming (evict-first) accesses to p, s, x vs plain accesses
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/r02d_cs_ab.txt
for rnd in 1 2; do
  timeout 600 python tools/scripts/r02d_cs_ab.py >> gpurun_out/r02d_cs_ab.txt 2>&1
  NPC_LIB_PATH=$GRAFT_REPO_ROOT/paper_2208_01339_b200/variants/libnpc_cg_nocs.so timeout 600 python tools/scripts/r02d_cs_ab.py >> gpurun_out/r02d_cs_ab.txt 2>&1
done
grep -v "rep 0" gpurun_out/r02d_cs_ab.txt
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pcg_branches.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
