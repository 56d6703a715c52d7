# final check of the driver's entry points: smoke(), the default bench line, the reference arm
cd $GRAFT_REPO_ROOT; R=gpurun_out/final; mkdir -p $R
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
( time python bench.py > $R/bench_default.json 2> $R/bench_default.err ) 2>&1 | grep real
python -c "import json;d=json.load(open('$R/bench_default.json'));print(round(d['value'],1), round(d['e2e']['value'],1), d['ms_per_step'], d['gpu_launches'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d['roofline']['traffic'], d['cpu_baseline']['value'], d['clocks'])"
( time python bench.py --impl reference --steps 2 --warmup 1 > $R/bench_reference.json 2> $R/bench_reference.err ) 2>&1 | grep real
cat $R/bench_reference.json | cut -c1-600
