# VF_LIBM_ASSUME A/B (argument-range assumptions for the inlined logf / expf)
python tools/kbench.py --images 256 --only exact > gpurun_out/kb0.log 2>&1
VF_LIB=paper_1009_0959_b200/libvf_as.so python tools/kbench.py --images 256 --only exact > gpurun_out/kb1.log 2>&1
python tools/dev/plan_stats_ab.py > gpurun_out/ab0.log 2>&1
VF_LIB=paper_1009_0959_b200/libvf_as.so python tools/dev/plan_stats_ab.py > gpurun_out/ab1.log 2>&1
VF_LIB=paper_1009_0959_b200/libvf_as.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/aspar.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stream or angular" > gpurun_out/defpar.log 2>&1
