# A/B of plans with and without statistics nodes (tools/dev/plan_stats_ab.py)
python tools/dev/plan_stats_ab.py > gpurun_out/ab0.log 2>&1
