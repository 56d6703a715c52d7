# A/B timing of library variants on a config: bash tools/gpu_ab.sh CONFIG variant...
# (variant "main" = paper_2103_09943_b200/lib/libfbmp_gpu.so, others lib/exp/libfbmp_gpu_<v>.so)
cd $GRAFT_REPO_ROOT
cfg=$1; shift
for v in "$@"; do
  if [ "$v" = main ]; then unset FBMP_GPU_LIB; else export FBMP_GPU_LIB=$PWD/paper_2103_09943_b200/lib/exp/libfbmp_gpu_$v.so; fi
  timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 10 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$cfg $v', round(d['ms_per_step'],3), {k:round(v['avg_ms']*1e3,1) for k,v in d['roofline']['cg_kernels'].items()}, d['iterations']['cg'][:8])" || tail -3 gpurun_out/ab_$v.err
done
unset FBMP_GPU_LIB
