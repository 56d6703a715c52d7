# Scratch driver for gpurun debugging sessions (overwritten freely): CG iteration counts and the
# HRMS difference to the golden fixtures on the C1 and C2 scenes for the current build.
cd $GRAFT_REPO_ROOT
TAG=c1 python tools/c1_iters.py C1 15
TAG=c2 python tools/c1_iters.py C2 17
