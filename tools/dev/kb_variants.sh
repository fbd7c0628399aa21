# dev scratch (round-2 tuning): A/B of library variants built with build.py --variant
# A/B timing of library variants (VARIANTS="main rn1 ..."; main = libvf.so) and,
# with CHECK=1, a parity check of each variant on a C2-size image first.
for v in ${VARIANTS:-main}; do
  if [ "$v" = "main" ]; then lib=paper_1009_0959_b200/libvf.so; else lib=paper_1009_0959_b200/libvf_$v.so; fi
  if [ -n "$CHECK" ]; then VF_LIB=$lib python -m pytest tests/test_gpu_parity.py -q -x -k "angular and (c2 or ragged or palette or branch)" 2>&1 | tail -1; fi
  VF_LIB=$lib python tools/kbench.py --images 256 --only ${ONLY:-angular/minimax}
done
