# multi-reference statistics node: tests + A/B against one node per reference
timeout 900 python -m pytest tests/test_gpu_plan_stats.py tests/test_gpu_debug_bounds.py tests/test_bench_contract.py -m gpu -q -x > gpurun_out/t.log 2>&1
python tools/dev/plan_stats_ab.py > gpurun_out/ab0.log 2>&1
VF_PLAN_STATS_SPLIT=1 python tools/dev/plan_stats_ab.py > gpurun_out/ab1.log 2>&1
