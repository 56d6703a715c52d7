cd $GRAFT_REPO_ROOT; R=gpurun_out/r02e; mkdir -p $R
timeout 1200 python -m pytest tests -m gpu -x -q > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
timeout 300 python bench.py --no-cpu-baseline > $R/bench_c2.json 2> $R/bench_c2.err
timeout 300 python bench.py --no-cpu-baseline --config C1 > $R/bench_c1.json 2> $R/bench_c1.err
bash tools/admm_prof.sh
tail -n 3 $R/gputest.log
