# Refresh the committed measurements (bench lines C1..C5, fp32 lines, C2 launch list, ncu capture of
# the CG kernels) into gpurun_out/refresh/; copy the ones to keep into profiles/.
cd $GRAFT_REPO_ROOT
R=gpurun_out/refresh; mkdir -p $R
timeout 400 python bench.py --config C2 > $R/bench_c2.json 2> $R/bench_c2.err
timeout 300 python bench.py --config C1 --steps 10 > $R/bench_c1.json 2> $R/bench_c1.err
timeout 400 python bench.py --config C3 --steps 5 --no-cpu-baseline > $R/bench_c3.json 2> $R/bench_c3.err
timeout 400 python bench.py --config C4 --steps 5 --no-cpu-baseline > $R/bench_c4.json 2> $R/bench_c4.err
timeout 600 python bench.py --config C5 --steps 3 --no-cpu-baseline > $R/bench_c5.json 2> $R/bench_c5.err
timeout 300 python bench.py --config C2 --precision 32 --no-cpu-baseline > $R/bench_c2_f32.json 2> $R/bench_c2_f32.err
timeout 600 python bench.py --config C5 --precision 32 --steps 3 --no-cpu-baseline > $R/bench_c5_f32.json 2> $R/bench_c5_f32.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file $R/launches_c2.csv python tools/run_one.py C2 2 > $R/ncu_launch.log 2>&1
# one chain (FBMP_CG_GROUPS=1), as in bench.py's profile pass: the launches cover all four channels
FBMP_CG_GROUPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_q3|k_du|k_llp2" --launch-skip 60 --launch-count 3 -o $R/cg_c2 -f python tools/run_one.py C2 1 > $R/ncu_full.log 2>&1
for c in c1 c2 c3 c4 c5 c2_f32 c5_f32; do python -c "import json;d=json.load(open('$R/bench_$c.json'));print('$c', round(d['value'],1), round(d['e2e']['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],3), {k:round(v['frac'],3) for k,v in d['roofline']['operators'].items()}, d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -2 $R/bench_$c.err; done
tail -1 $R/ncu_full.log
