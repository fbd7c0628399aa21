cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python tools/kbench.py C2 C4 C3 2>&1 | tail -5
python tools/prof_driver.py --config C4 > /dev/null && timeout 600 ncu --set full --import-source on --clock-control none -k regex:vf_ -s 7 -c 7 -o gpurun_out/prof_C4b python tools/prof_driver.py --config C4 > gpurun_out/ncu_C4b.log 2>&1; tail -2 gpurun_out/ncu_C4b.log
