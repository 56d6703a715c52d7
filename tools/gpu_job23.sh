cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/env
run() { # name, env...
  name=$1; shift
  env "$@" timeout 300 python bench.py --config C2 --no-cpu-baseline --steps 10 > gpurun_out/env/$name.json 2>gpurun_out/env/$name.err
  python -c "import json;d=json.load(open('gpurun_out/env/$name.json'));print('$name', round(d['value'],1), round(d['ms_per_step'],3), {k:round(x*1e3,1) for k,x in d['roofline']['kernel_avg_ms'].items()}, d['iterations']['cg'][:8])" || tail -3 gpurun_out/env/$name.err
}
run base FOO=1
run pdl5 FBMP_PDL=5
run pdl3 FBMP_PDL=3
run pdl6 FBMP_PDL=6
run pdl0 FBMP_PDL=0
run sr8 FBMP_KQ3_SR=8
run sr13 FBMP_KQ3_SR=13
run sr16 FBMP_KQ3_SR=16
run grp2 FBMP_CG_GROUPS=2
