# dev scratch (round-2 tuning): A/B of library variants built with build.py --variant
# step-time A/B of library variants: VARIANTS="main f24 ..." (main = libvf.so)
for v in ${VARIANTS:-main}; do
  if [ "$v" = "main" ]; then lib=paper_1009_0959_b200/libvf.so; else lib=paper_1009_0959_b200/libvf_$v.so; fi
  VF_LIB=$lib python bench.py --steps 10 --warmup 3 --no-c3 --no-paper --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/step_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/step_$v.json')); print('$v', round(d['value']), round(d['ms_per_step'], 3))"
done
