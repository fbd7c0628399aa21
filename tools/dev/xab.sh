# C2: fused exp/log node for small plans (VF_PLAN_FUSE=2) vs one node per filter
B="python bench.py --workload c2 --steps 200 --warmup 20 --no-cpu-baseline --no-paper --no-e2e"
$B > gpurun_out/c2_default.json 2>/dev/null
VF_PLAN_FUSE=2 $B > gpurun_out/c2_fuse4.json 2>/dev/null
VF_LIB=paper_1009_0959_b200/libvf_n8.so VF_PLAN_FUSE=2 $B > gpurun_out/c2_fuse8.json 2>/dev/null
$B > gpurun_out/c2_default2.json 2>/dev/null
