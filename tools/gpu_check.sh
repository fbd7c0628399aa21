#!/bin/bash
# one gpurun call: build check, GPU tests, smoke, bench, then (only if the plain
# bench exited 0) the ncu launch list of the same bench command.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import paper_1009_0959_b200 as p; p.load_library()" || python -m paper_1009_0959_b200.build
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
BENCH="python bench.py --steps ${STEPS:-20} --warmup 3 ${BENCH_ARGS:-}"
timeout 600 $BENCH > gpurun_out/bench.json 2> gpurun_out/bench.err; rc=$?; echo "bench exit $rc" >> gpurun_out/bench.err
if [ $rc -eq 0 ] && [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     $BENCH > gpurun_out/ncu_launch.log 2>&1
  echo "ncu exit $?" >> gpurun_out/ncu_launch.log
fi
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench.json | head -c 3000; tail -2 gpurun_out/bench.err
