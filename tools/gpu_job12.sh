cd $GRAFT_REPO_ROOT; R=gpurun_out/r02k; mkdir -p $R
timeout 1500 python -m pytest tests -m gpu -x -q > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
timeout 300 python bench.py > $R/bench_c2.json 2> $R/bench_c2.err
timeout 300 python bench.py --config C1 --steps 10 > $R/bench_c1.json 2> $R/bench_c1.err
timeout 400 python bench.py --config C3 --steps 5 > $R/bench_c3.json 2> $R/bench_c3.err
timeout 400 python bench.py --config C4 --steps 5 --no-cpu-baseline > $R/bench_c4.json 2> $R/bench_c4.err
for U in 2 4; do FBMP_GPU_LIB=paper_2103_09943_b200/lib/exp/libfbmp_gpu_klu$U.so timeout 300 python bench.py --no-cpu-baseline > $R/bench_c2_klu$U.json 2> $R/bench_c2_klu$U.err; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_guided3" --launch-count 1 -o $R/gf python tools/run_one.py C2 1 > $R/ncu_gf.log 2>&1
tail -n 3 $R/gputest.log
