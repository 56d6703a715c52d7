cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
for c in C4 C3 C5; do timeout 400 python bench.py --config $c --no-cpu-baseline --steps 5 > gpurun_out/q3_$c.json 2>gpurun_out/q3_$c.err; python -c "import json;d=json.load(open('gpurun_out/q3_$c.json'));print('$c', round(d['ms_per_step'],3), d['value'], {k:round(v['avg_ms']*1e3,1) for k,v in d['roofline']['cg_kernels'].items()})"; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_dterm|k_llp2" --launch-skip 40 --launch-count 2 -o gpurun_out/kdl python tools/run_one.py C2 1 > gpurun_out/ncu_kdl.log 2>&1
tail -2 gpurun_out/ncu_kdl.log
