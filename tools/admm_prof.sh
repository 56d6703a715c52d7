# Phase breakdown of k_admm (clock64 of CTA 0, summed over the iterations): x/y-step, z mat-vec,
# finite check, simplex projection, {u,p} anchor, {u,p} solve, multipliers + norms.
cd $GRAFT_REPO_ROOT; R=gpurun_out/admm; mkdir -p $R
for c in C1 C2 C5; do FBMP_GPU_LIB=paper_2103_09943_b200/lib/exp/libfbmp_gpu_aprof.so timeout 300 python tools/run_one.py $c 2 > $R/prof_$c.log 2>&1; done
tail -n 4 $R/prof_*.log
