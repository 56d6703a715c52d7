cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/env
run() { # name, config, steps, env...
  name=$1; cfg=$2; st=$3; shift; shift; shift
  env "$@" timeout 400 python bench.py --config $cfg --no-cpu-baseline --steps $st > gpurun_out/env/$name.json 2>gpurun_out/env/$name.err
  python -c "import json;d=json.load(open('gpurun_out/env/$name.json'));print('$name', round(d['value'],1), round(d['ms_per_step'],3), d['iterations']['cg'][:8], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/env/$name.err
}
run c2_base C2 10 FOO=1
run c2_sr13 C2 10 FBMP_KQ3_SR=13
run c2_sr16 C2 10 FBMP_KQ3_SR=16
run c2_sr20 C2 10 FBMP_KQ3_SR=20
run c2_sr8 C2 10 FBMP_KQ3_SR=8
