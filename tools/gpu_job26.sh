cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/env
run() { # name, config, steps, env...
  name=$1; cfg=$2; st=$3; shift; shift; shift
  env "$@" timeout 400 python bench.py --config $cfg --no-cpu-baseline --steps $st > gpurun_out/env/$name.json 2>gpurun_out/env/$name.err
  python -c "import json;d=json.load(open('gpurun_out/env/$name.json'));print('$name', round(d['value'],1), round(d['ms_per_step'],3), d['iterations']['cg'][:8], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/env/$name.err
}
run c2_g2 C2 10 FOO=1
run c2_g3 C2 10 FBMP_CG_GROUPS=3
run c2_g4 C2 10 FBMP_CG_GROUPS=4
run c3_g2 C3 5 FOO=1
run c3_g4 C3 5 FBMP_CG_GROUPS=4
run c5_g2 C5 2 FOO=1
run c5_g4 C5 2 FBMP_CG_GROUPS=4
run c1_g2 C1 10 FOO=1
run c1_g4 C1 10 FBMP_CG_GROUPS=4
