#!/bin/bash
# Round evidence: GPU tests, smoke, default bench (plain), the ncu launch list of
# the same bench command, and one `ncu --set full` capture of every filter kernel
# (C2 = the bench workload, C4 = throughput regime).  Results in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
BENCH="python bench.py"
timeout 900 $BENCH > gpurun_out/bench.json 2> gpurun_out/bench.err; rc=$?; echo "bench exit $rc" >> gpurun_out/bench.err
for c in C3 C4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
if [ $rc -eq 0 ]; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $BENCH > gpurun_out/ncu_launch.log 2>&1
  echo "ncu launch exit $?" >> gpurun_out/ncu_launch.log
  python tools/prof_driver.py --config C2 > /dev/null && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:vf_ -s 7 -c 7 -o gpurun_out/prof_C2 python tools/prof_driver.py --config C2 > gpurun_out/ncu_C2.log 2>&1
  python tools/prof_driver.py --config C4 > /dev/null && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:vf_ -s 7 -c 7 -o gpurun_out/prof_C4 python tools/prof_driver.py --config C4 > gpurun_out/ncu_C4.log 2>&1
  python tools/prof_driver.py --config C3 --rounds 1 > /dev/null && \
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:vf_ -s 7 -c 7 -o gpurun_out/prof_C3 python tools/prof_driver.py --config C3 > gpurun_out/ncu_C3.log 2>&1
fi
# summarise on the box (the .ncu-rep files exceed gpurun's 64 MiB copy-back limit), keep the C4 report only
mkdir -p gpurun_out/prof_summary
for c in C2 C3 C4; do
  [ -f gpurun_out/prof_$c.ncu-rep ] && python tools/ncu_source_summary.py gpurun_out/prof_$c.ncu-rep > gpurun_out/prof_summary/${TAG:-r01}_sass_mix_$c.txt 2>&1
done
VF_PROF_DIR=gpurun_out/prof_summary python tools/summarize_round.py ${TAG:-r01} > /dev/null 2>&1
rm -f gpurun_out/prof_C2.ncu-rep gpurun_out/prof_C3.ncu-rep
du -sh gpurun_out
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/bench.err; tail -1 gpurun_out/ncu_launch.log
