# A/B timing of library variants: bash tools/gpu_ab.sh "C2 C5" variant...
# (variant "main" = paper_2103_09943_b200/lib/libfbmp_gpu.so, others lib/exp/libfbmp_gpu_<v>.so)
cd $GRAFT_REPO_ROOT
cfgs=$1; shift
mkdir -p gpurun_out/ab
for v in "$@"; do
  if [ "$v" = main ]; then unset FBMP_GPU_LIB; else export FBMP_GPU_LIB=$PWD/paper_2103_09943_b200/lib/exp/libfbmp_gpu_$v.so; fi
  for c in $cfgs; do
  st=10; [ "$c" = C5 ] && st=3
  timeout 400 python bench.py --config $c --no-cpu-baseline --steps $st > gpurun_out/ab/${c}_$v.json 2>gpurun_out/ab/${c}_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab/${c}_$v.json'));print('$c $v', round(d['value'],1), round(d['ms_per_step'],3), {k:round(x*1e3,1) for k,x in d['roofline']['kernel_avg_ms'].items()}, d['iterations']['cg'][:8], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab/${c}_$v.err
  done
done
unset FBMP_GPU_LIB
