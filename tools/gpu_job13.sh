cd $GRAFT_REPO_ROOT; R=gpurun_out/r02l; mkdir -p $R
timeout 600 python -m pytest tests/test_gpu_fp32.py -x -q > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
timeout 300 python bench.py --no-cpu-baseline --precision 32 > $R/bench_c2_f32.json 2> $R/bench_c2_f32.err
FBMP_KL_NOQUAD=1 timeout 300 python bench.py --no-cpu-baseline --precision 32 > $R/bench_c2_f32_noquad.json 2> $R/bench_c2_f32_noquad.err
timeout 300 python bench.py --no-cpu-baseline --precision 32 --config C5 --steps 2 > $R/bench_c5_f32.json 2> $R/bench_c5_f32.err
FBMP_KL1=1 timeout 300 python bench.py --no-cpu-baseline --config C1 --steps 10 > $R/bench_c1_kl1.json 2> $R/bench_c1_kl1.err
FBMP_KL1=1 timeout 600 python -m pytest tests/test_gpu_pipeline.py -x -q -k "golden_c1 or blind_c1" > $R/gputest_kl1.log 2>&1; echo pytest=$? >> $R/gputest_kl1.log
tail -n 3 $R/gputest.log
