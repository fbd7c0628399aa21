# quick GPU iteration: GPU tests (or a subset via PYTEST_K), per-kernel timings, optional tile sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -8
timeout 300 python tools/kbench.py ${KB_CONFIGS:-C2 C4 C3} 2>&1 | tail -5
[ -n "$TUNE" ] && timeout 600 bash tools/tune_tiles.sh 2>&1 | tail -20
true
