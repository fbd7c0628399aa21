# dev scratch: the bench's per_node times for library variants (VARIANTS="main b16 ...")
for v in ${VARIANTS:-main}; do
  if [ "$v" = "main" ]; then lib=paper_1009_0959_b200/libvf.so; else lib=paper_1009_0959_b200/libvf_$v.so; fi
  VF_LIB=$lib python bench.py --steps 10 --warmup 3 --no-c3 --no-paper --no-cpu-baseline --no-e2e > gpurun_out/node_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/node_$v.json')); print('$v', round(d['ms_per_step'], 3), {k: round(x['ms'], 3) for k, x in d['per_node'].items()})"
done
