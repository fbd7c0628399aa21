# the VF_EXACT_LIBM=1 build: parity test + the whole default bench under it
timeout 900 python -m pytest tests/test_gpu_exact_libm.py -m gpu -q -x > gpurun_out/t.log 2>&1
VF_LIB=paper_1009_0959_b200/libvf_paperlibm.so timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_paperlibm.json 2> gpurun_out/bench_paperlibm.err
VF_LIB=paper_1009_0959_b200/libvf_paperlibm.so timeout 600 python bench.py --workload c2 --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2_paperlibm.json 2>/dev/null
