#!/bin/bash
# Round-2 evidence, second call: ncu --set full of the C3 5x5 kernels (role-sum
# angular kernels, 5x5 exp/log window kernels) and the statistics passes.
# Afterwards, here:
#   python tools/ncu_full_summary.py gpurun_out/r02_full_c3_raw.csv > profiles/r02_ncu_full_c3.md
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PROF_IMAGES=64 timeout 1500 ncu --set full --clock-control none --kernel-name-base mangled \
  -k 'regex:role_kernelILi5|el_kernelILi5|stats_multi' -c 14 -f \
  -o gpurun_out/r02_full_c3 python tools/prof_kernels.py > gpurun_out/ncu_full_c3.log 2>&1
echo "ncu full c3 exit $?" >> gpurun_out/ncu_full_c3.log
ncu -i gpurun_out/r02_full_c3.ncu-rep --page raw --csv > gpurun_out/r02_full_c3_raw.csv 2>> gpurun_out/ncu_full_c3.log
# the report itself (12 launches with source) is over gpurun's 64 MiB return limit: keep the raw page only
rm -f gpurun_out/r02_full_c3.ncu-rep
tail -3 gpurun_out/ncu_full_c3.log; wc -l gpurun_out/r02_full_c3_raw.csv
