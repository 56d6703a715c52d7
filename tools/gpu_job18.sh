cd $GRAFT_REPO_ROOT; R=gpurun_out/r02q; mkdir -p $R
timeout 300 python bench.py --no-cpu-baseline > $R/bench_c2_du.json 2> $R/bench_c2_du.err
FBMP_DU=0 timeout 300 python bench.py --no-cpu-baseline > $R/bench_c2_nodu.json 2> $R/bench_c2_nodu.err
for f in du nodu; do python -c "import json;d=json.load(open('$R/bench_c2_$f.json'));print('$f', round(d['value'],1), d['ms_per_step'], d['stages_ms'], d['roofline']['kernel_avg_ms'], d['iterations'])" || tail -5 $R/bench_c2_$f.err; done
timeout 1500 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_fp32.py -m gpu -x -q > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
tail -n 15 $R/gputest.log
