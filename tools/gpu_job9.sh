cd $GRAFT_REPO_ROOT; R=gpurun_out/r02h; mkdir -p $R
timeout 600 python -m pytest tests/test_gpu_fp32.py -x -q > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
timeout 300 python bench.py --no-cpu-baseline --precision 32 > $R/bench_c2_f32.json 2> $R/bench_c2_f32.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 1600 --csv --log-file $R/launches_c1.csv python tools/run_one.py C1 2 > $R/ncu_launch_c1.log 2>&1
tail -n 3 $R/gputest.log
