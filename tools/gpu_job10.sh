cd $GRAFT_REPO_ROOT; R=gpurun_out/r02i; mkdir -p $R
timeout 300 python bench.py --no-cpu-baseline > $R/bench_c2_kl5.json 2> $R/bench_c2_kl5.err
FBMP_KL=2 timeout 300 python bench.py --no-cpu-baseline > $R/bench_c2_kl2.json 2> $R/bench_c2_kl2.err
timeout 1200 python -m pytest tests/test_gpu_ops.py tests/test_gpu_pipeline.py tests/test_gpu_fp32.py -x -q > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
timeout 300 python bench.py --no-cpu-baseline --precision 32 > $R/bench_c2_f32_kl5.json 2> $R/bench_c2_f32_kl5.err
timeout 600 python bench.py --config C5 --steps 2 --no-cpu-baseline > $R/bench_c5_kl5.json 2> $R/bench_c5_kl5.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_llp5" --launch-skip 20 --launch-count 1 -o $R/kl5 python tools/run_one.py C2 1 > $R/ncu_kl5.log 2>&1
tail -n 3 $R/gputest.log
