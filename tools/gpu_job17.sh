cd $GRAFT_REPO_ROOT; R=gpurun_out/r02p; mkdir -p $R
timeout 1800 python -m pytest tests -m gpu -x -q > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
timeout 400 python bench.py > $R/bench_c2.json 2> $R/bench_c2.err
tail -n 3 $R/gputest.log; cat $R/bench_c2.json
