# exact variants (expm1f / log1pf): rows per thread of the single-filter kernels
for o in 2 4; do VF_EL_OPT=$o python tools/kbench.py --images 256 --only exact > gpurun_out/kb_opt$o.log 2>&1; done
python tools/dev/plan_stats_ab.py > gpurun_out/ab0.log 2>&1
