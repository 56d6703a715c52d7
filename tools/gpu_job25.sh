cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/env
run() { # name, config, steps, env...
  name=$1; cfg=$2; st=$3; shift; shift; shift
  env "$@" timeout 400 python bench.py --config $cfg --no-cpu-baseline --steps $st > gpurun_out/env/$name.json 2>gpurun_out/env/$name.err
  python -c "import json;d=json.load(open('gpurun_out/env/$name.json'));print('$name', round(d['value'],1), round(d['ms_per_step'],3), d['iterations']['cg'][:8], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/env/$name.err
}
run c2_def C2 10 FOO=1
run c2_du1 C2 10 FBMP_DU_PER_SM=1
run c3_def C3 5 FOO=1
run c3_du1 C3 5 FBMP_DU_PER_SM=1
run c5_def C5 2 FOO=1
run c5_du1 C5 2 FBMP_DU_PER_SM=1
run c4_def C4 3 FOO=1
run c1_def C1 10 FOO=1
timeout 300 python bench.py --config C2 --precision 32 --no-cpu-baseline --steps 10 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c2_f32', round(d['value'],1), d['ms_per_step'])"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/env/gputest.log 2>&1; echo pytest=$? >> gpurun_out/env/gputest.log
tail -n 4 gpurun_out/env/gputest.log
