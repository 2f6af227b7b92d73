cd $GRAFT_REPO_ROOT
V=paper_2208_01339_b200/variants
L=paper_2208_01339_b200/libnpc.so
for reps in 10 300; do
AB_INTERVAL=17.6:144820 timeout 900 python tools/ab_variants.py --config 3 --k 50 --reps $reps --libs $L,$V/libnpc_nozwin.so,$L,$V/libnpc_nozwin.so 2>&1 | cut -c1-150
done
