cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python tools/kbench.py C2 C4 C3 2>&1 | tail -5
