#!/bin/bash
# GPU tests + short benches of C2/C3/C4 (no cpu baseline/e2e), summaries to stdout
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} 2>&1 | tail -${PYTEST_TAIL:-4}
for c in ${CONFIGS:-C2 C3 C4}; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err || tail -3 gpurun_out/bench_$c.err
done
