#!/bin/bash
# Round-2 evidence in one gpurun call: GPU tests + smoke, per-kernel ncu pipe
# metrics (-> profiles/ncu_exec.json on the box, so the bench attaches them),
# the default bench, the C2 bench, the bench's ncu launch list, and ncu
# --set full of the step's dominant node.  Afterwards, here:
#   cp gpurun_out/ncu_exec.json profiles/; tail -1 gpurun_out/bench.json > profiles/r02_bench_C4.json; ...
#   python tools/ncu_launches.py gpurun_out/launches.csv --step el_fused5_kernel:1 \
#     stream_kernelILi1ELi2ELi32:1 stream_kernelILi1ELi2ELi16:1 stats_multi_kernelILi1ELi4:2 \
#     stats_multi_kernelILi2ELi4:1 stats_finalize:1 > profiles/r02_launches_summary.md
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{ nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; nproc; } > gpurun_out/box.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 ncu --metrics $(python tools/ncu_exec.py --metrics) --clock-control none --print-kernel-base mangled --csv \
  --log-file gpurun_out/exec.csv python tools/prof_kernels.py > gpurun_out/ncu_exec.log 2>&1
echo "ncu exec exit $?" >> gpurun_out/ncu_exec.log
python tools/ncu_exec.py gpurun_out/exec.csv >> gpurun_out/ncu_exec.log 2>&1 && cp profiles/ncu_exec.json gpurun_out/ncu_exec.json
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 600 python bench.py --workload c2 --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --print-kernel-base mangled --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch exit $?" >> gpurun_out/ncu_launch.log
PROF_IMAGES=256 timeout 1200 ncu --set full --clock-control none -k 'regex:fused5' -c 1 \
  -o gpurun_out/r02_full python tools/prof_kernels.py > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ncu_full.log
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; tail -1 gpurun_out/bench.err
