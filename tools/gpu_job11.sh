cd $GRAFT_REPO_ROOT; R=gpurun_out/r02j; mkdir -p $R
./tools/fp_peak > $R/fp_peak.json 2>&1
timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -k "guided" > $R/gputest_ops.log 2>&1; echo pytest=$? >> $R/gputest_ops.log
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q -k "golden or blind_c1 or strips_nccl or batch" > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
timeout 300 python bench.py --no-cpu-baseline > $R/bench_c2.json 2> $R/bench_c2.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_guided3" --launch-count 1 -o $R/gf python tools/run_one.py C2 1 > $R/ncu_gf.log 2>&1
tail -n 3 $R/gputest.log
