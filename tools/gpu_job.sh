# scratch GPU job: bench lines of the configs given (default "C2"), then the named pytest selection
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/job
for c in ${CFGS:-C2}; do
  st=10; [ "$c" = C5 ] && st=3; [ "$c" = C4 ] && st=3
  timeout 400 python bench.py --config $c --no-cpu-baseline --steps $st > gpurun_out/job/$c.json 2>gpurun_out/job/$c.err
  python -c "import json;d=json.load(open('gpurun_out/job/$c.json'));print('$c', round(d['value'],1), round(d['ms_per_step'],3), {k:round(x*1e3,1) for k,x in d['roofline']['kernel_avg_ms'].items()}, d['iterations']['cg'][:8], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/job/$c.err
done
if [ -n "$TESTS" ]; then timeout 1800 python -m pytest $TESTS -m gpu -x -q > gpurun_out/job/gputest.log 2>&1; echo pytest=$? >> gpurun_out/job/gputest.log; tail -n 4 gpurun_out/job/gputest.log; fi
