cd $GRAFT_REPO_ROOT; R=gpurun_out/r02r; mkdir -p $R
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_du" --launch-skip 20 --launch-count 1 -o $R/du_c2 -f python tools/run_one.py C2 1 > $R/ncu_full.log 2>&1
tail -1 $R/ncu_full.log
