#!/bin/bash
# Functional check of bench.py's N > 1 code paths on a 1-GPU box: N ranks
# share the device over gloo (VF_BENCH_BACKEND=gloo).  Timings are not
# measurements (the ranks share one GPU); exit codes and the JSON lines are
# what this checks.  The driver's N > 1 runs use NCCL, one rank per GPU.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export VF_BENCH_BACKEND=gloo PYTHONFAULTHANDLER=1
: > gpurun_out/n_summary.txt
for n in ${RANKS:-2 4}; do
  for wl in c4 c5; do
    extra=""; [ $wl = c4 ] && extra="--images 64 --no-c3 --no-paper"
    timeout -s INT 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + n)) bench.py --gpus $n --workload $wl --steps 3 --warmup 3 $extra \
      > gpurun_out/n${n}_$wl.json 2> gpurun_out/n${n}_$wl.err
    echo "$wl n=$n exit $?" >> gpurun_out/n_summary.txt
  done
done
cat gpurun_out/n_summary.txt
