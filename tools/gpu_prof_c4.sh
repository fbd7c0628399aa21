# GPU tests, then ncu --set full of the C4 filter kernels (second round of launches)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -4
python tools/prof_driver.py --config ${CFG:-C4} > /dev/null && timeout 600 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-vf_} -s ${SKIP:-7} -c ${COUNT:-7} -o gpurun_out/prof_${TAG:-C4b} python tools/prof_driver.py --config ${CFG:-C4} > gpurun_out/ncu_${TAG:-C4b}.log 2>&1; tail -2 gpurun_out/ncu_${TAG:-C4b}.log
