cd $GRAFT_REPO_ROOT
NPC_CREATE_TIMES=1 timeout 600 python tools/create_times.py --configs 3 2>&1 | tail -20
nproc
