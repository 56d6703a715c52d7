cd $GRAFT_REPO_ROOT; R=gpurun_out/r02n; mkdir -p $R
for CS in 4 8 16; do FBMP_ADMM_CLUSTER=$CS timeout 300 python tools/run_one.py C2 3 > $R/c2_cs$CS.log 2>&1; FBMP_ADMM_CLUSTER=$CS timeout 300 python tools/run_one.py C1 3 > $R/c1_cs$CS.log 2>&1; FBMP_ADMM_CLUSTER=$CS timeout 300 python tools/run_one.py C5 2 > $R/c5_cs$CS.log 2>&1; done
tail -n 1 $R/*.log
