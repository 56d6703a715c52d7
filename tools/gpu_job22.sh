cd $GRAFT_REPO_ROOT; R=gpurun_out/r02u; mkdir -p $R
for v in main nst2; do
  if [ "$v" = main ]; then unset FBMP_GPU_LIB; else export FBMP_GPU_LIB=$PWD/paper_2103_09943_b200/lib/exp/libfbmp_gpu_$v.so; fi
  for c in C2 C5; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --steps 5 > $R/ab_${c}_$v.json 2>$R/ab_${c}_$v.err
  python -c "import json;d=json.load(open('$R/ab_${c}_$v.json'));print('$c $v', round(d['value'],1), round(d['ms_per_step'],3), d['roofline']['kernel_avg_ms'])" || tail -3 $R/ab_${c}_$v.err
  done
done
unset FBMP_GPU_LIB
timeout 1800 python -m pytest tests -m gpu -x -q > $R/gputest.log 2>&1; echo pytest=$? >> $R/gputest.log
tail -n 4 $R/gputest.log
