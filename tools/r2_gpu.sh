#!/bin/bash
# One gpurun call: box facts, GPU tests (PYTEST_K selects), smoke (SMOKE=1),
# the default bench (BENCH_ARGS), optional ncu launch list (NCU=1).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{ nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; nproc; free -g; } > gpurun_out/box.txt 2>&1
if [ -n "$PYTEST_K" ]; then
  timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
elif [ -z "$NO_PYTEST" ]; then
  timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
if [ -n "$SMOKE" ]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
fi
if [ -z "$NO_BENCH" ]; then
  BENCH="python bench.py --steps ${STEPS:-20} --warmup ${WARMUP:-5} ${BENCH_ARGS:-}"
  timeout 900 $BENCH > gpurun_out/bench.json 2> gpurun_out/bench.err; rc=$?; echo "bench exit $rc" >> gpurun_out/bench.err
  if [ $rc -eq 0 ] && [ -n "$NCU" ]; then
    timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --print-kernel-base mangled --csv \
       --log-file gpurun_out/launches.csv $BENCH --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
    echo "ncu exit $?" >> gpurun_out/ncu_launch.log
  fi
fi
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > gpurun_out/extra.log 2>&1; echo "extra exit $?" >> gpurun_out/extra.log; fi
cat gpurun_out/box.txt; tail -5 gpurun_out/pytest_gpu.log 2>/dev/null; tail -2 gpurun_out/smoke.log 2>/dev/null
head -c 1500 gpurun_out/bench.json 2>/dev/null; echo; tail -3 gpurun_out/bench.err 2>/dev/null; tail -5 gpurun_out/extra.log 2>/dev/null
