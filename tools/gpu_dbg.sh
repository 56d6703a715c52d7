cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_q3 --launch-skip 20 --launch-count 1 -o gpurun_out/kq3b python tools/run_one.py C2 1 > gpurun_out/ncu_kq3b.log 2>&1
tail -1 gpurun_out/ncu_kq3b.log
