# final bench (ncu_exec.json of this library committed: traffic + per-kernel ncu records attach) + ncu --set full of the angular streamed kernels
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
PROF_IMAGES=256 timeout 1200 ncu --set full --clock-control none -k regex:vf_angular_stream_kernel -c 6 \
  -o gpurun_out/r02_full_ang python tools/prof_kernels.py > gpurun_out/ncu_full_ang.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full_ang.log
