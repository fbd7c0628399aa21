# dev scratch (round-2 tuning): A/B of library variants built with build.py --variant
run() { env "$@" python bench.py --workload c2 --steps 300 --warmup 5 --no-cpu-baseline --no-paper --no-e2e > gpurun_out/c2x.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/c2x.json')); print('$*', round(d['ms_per_step']*1e3,2), {k: round(v['ms']*1e3,1) for k, v in d['per_kernel'].items()})"; }
run X=1
run VF_EL_OPT=2
run VF_EL_OPT=4
run VF_SHARED_PPT=1
run VF_SHARED_PPT=2
