cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/env
run() { # name, config, steps, env...
  name=$1; cfg=$2; st=$3; shift; shift; shift
  env "$@" timeout 400 python bench.py --config $cfg --no-cpu-baseline --steps $st > gpurun_out/env/$name.json 2>gpurun_out/env/$name.err
  python -c "import json;d=json.load(open('gpurun_out/env/$name.json'));print('$name', round(d['value'],1), round(d['ms_per_step'],3), {k:round(x*1e3,1) for k,x in d['roofline']['kernel_avg_ms'].items()}, d['iterations']['cg'][:8], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/env/$name.err
}
run c2 C2 10 FOO=1
run c3 C3 5 FOO=1
run c5 C5 2 FOO=1
timeout 900 python -m pytest tests/test_gpu_pipeline.py -m gpu -x -q -k "golden or c1 or c2 or batch or subset" > gpurun_out/env/gputest.log 2>&1; tail -n 3 gpurun_out/env/gputest.log
