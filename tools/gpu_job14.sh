cd $GRAFT_REPO_ROOT; R=gpurun_out/r02m; mkdir -p $R
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_shim.py tests/test_cli.py tests/test_gpu_fp32.py -x -q > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
timeout 300 python bench.py --no-cpu-baseline > $R/bench_c2.json 2> $R/bench_c2.err
timeout 300 python bench.py --no-cpu-baseline --config C3 --steps 5 > $R/bench_c3.json 2> $R/bench_c3.err
tail -n 3 $R/gputest.log
