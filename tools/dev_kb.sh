for v in ${VARIANTS:-"" a0}; do
  if [ "$v" = "main" ]; then python tools/kbench.py --images 256 --only angular/minimax; else VF_LIB=paper_1009_0959_b200/libvf_$v.so python tools/kbench.py --images 256 --only angular/minimax; fi
done
