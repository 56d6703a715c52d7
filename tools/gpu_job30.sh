cd $GRAFT_REPO_ROOT; R=gpurun_out/refresh; mkdir -p $R
FBMP_CG_GROUPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_q3|k_du|k_llp2" --launch-skip 60 --launch-count 3 -o $R/cg_c2_g1 -f python tools/run_one.py C2 1 > $R/ncu_full_g1.log 2>&1
tail -1 $R/ncu_full_g1.log
