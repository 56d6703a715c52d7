cd $GRAFT_REPO_ROOT; R=gpurun_out/r02d; mkdir -p $R
timeout 600 python -m pytest tests/test_gpu_fp32.py tests/test_gpu_ops.py -x -q > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
timeout 300 python bench.py --no-cpu-baseline > $R/bench_c2.json 2> $R/bench_c2.err
timeout 300 python bench.py --no-cpu-baseline --precision 32 > $R/bench_c2_f32.json 2> $R/bench_c2_f32.err
timeout 300 python bench.py --no-cpu-baseline --precision 32 --config C1 > $R/bench_c1_f32.json 2> $R/bench_c1_f32.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_guided2" --launch-count 1 -o $R/post python tools/run_one.py C2 1 > $R/ncu_post.log 2>&1
tail -n 5 $R/gputest.log
