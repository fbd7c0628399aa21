# exp/log tuning after the expf / logf exact variants
for o in 1 2 4; do VF_EL_OPT=$o python tools/kbench.py --images 256 --only exact > gpurun_out/kb_opt$o.log 2>&1; done
python tools/dev/plan_stats_ab.py > gpurun_out/ab_base.log 2>&1
for n in m2 m4 o1; do VF_LIB=paper_1009_0959_b200/libvf_$n.so python tools/dev/plan_stats_ab.py > gpurun_out/ab_$n.log 2>&1; done
