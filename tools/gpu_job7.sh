cd $GRAFT_REPO_ROOT; R=gpurun_out/r02f; mkdir -p $R
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_shim.py tests/test_gpu_pipeline.py -x -q -k "gram or solve_z or shim or golden or kernel or blind_c1" > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
timeout 300 python bench.py --no-cpu-baseline > $R/bench_c2.json 2> $R/bench_c2.err
bash tools/admm_prof.sh
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_gram_T2|k_admm" --launch-count 2 -o $R/fit python tools/run_one.py C2 1 > $R/ncu_fit.log 2>&1
tail -n 3 $R/gputest.log
