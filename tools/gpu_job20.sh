cd $GRAFT_REPO_ROOT; R=gpurun_out/r02s; mkdir -p $R
for c in C5 C3 C4; do
timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline > $R/bench_${c}_du.json 2> $R/bench_${c}_du.err
FBMP_DU=0 timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline > $R/bench_${c}_nodu.json 2> $R/bench_${c}_nodu.err
for f in du nodu; do python -c "import json;d=json.load(open('$R/bench_${c}_$f.json'));print('$c $f', round(d['value'],1), d['ms_per_step'], d['stages_ms'], d['roofline']['kernel_avg_ms'], d['iterations'])" || tail -5 $R/bench_${c}_$f.err; done
done
