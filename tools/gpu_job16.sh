cd $GRAFT_REPO_ROOT; R=gpurun_out/r02o; mkdir -p $R
timeout 1500 python -m pytest tests -m gpu -x -q > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
timeout 300 python bench.py --no-cpu-baseline > $R/bench_c2.json 2> $R/bench_c2.err
timeout 300 python bench.py --no-cpu-baseline --config C5 --steps 2 > $R/bench_c5.json 2> $R/bench_c5.err
tail -n 3 $R/gputest.log
