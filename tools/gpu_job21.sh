cd $GRAFT_REPO_ROOT; R=gpurun_out/r02t; mkdir -p $R
for c in C2 C5; do
timeout 600 python bench.py --config $c --steps 5 --no-cpu-baseline > $R/bench_${c}_du.json 2> $R/bench_${c}_du.err
python -c "import json;d=json.load(open('$R/bench_${c}_du.json'));print('$c du', round(d['value'],1), d['ms_per_step'], d['stages_ms'], d['roofline']['kernel_avg_ms'], d['iterations'])" || tail -5 $R/bench_${c}_du.err
done
timeout 600 python -m pytest tests/test_gpu_pipeline.py -m gpu -x -q -k "c1 or c2 or batch or subset or golden" > $R/gputest.log 2>&1; tail -3 $R/gputest.log
