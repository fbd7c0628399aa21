for p in 1 2 3; do echo "PPT=$p"; VF_SHARED_PPT=$p python tools/kbench.py C2 C4 C3 --only angular; done
for o in 1 2 4; do echo "OPT=$o"; VF_EL_OPT=$o python tools/kbench.py C2 C4; done
