for p in 1 2 3 4; do echo "PPT=$p"; VF_SHARED_PPT=$p python tools/kbench.py C2 C4 C3 --only angular; done
for o in 1 2 4; do echo "OPT=$o TMA"; VF_EL_OPT=$o python tools/kbench.py C2 C4; done
for o in 1 2 4; do echo "OPT=$o no TMA"; VF_NO_TMA=1 VF_EL_OPT=$o python tools/kbench.py C2 C4; done
echo "5x5 no TMA"; VF_NO_TMA=1 python tools/kbench.py C3
