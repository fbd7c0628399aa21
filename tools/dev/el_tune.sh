cd "$(dirname "$0")/../.."
for o in 2 4; do echo "OPT=$o TMA"; VF_EL_OPT=$o python tools/kbench.py C4 --only m; done
for o in 2 4; do echo "OPT=$o no TMA"; VF_NO_TMA=1 VF_EL_OPT=$o python tools/kbench.py C4 --only m; done
for mb in 5 3; do echo "minb OPT4 = $mb"; VF_LIB=tools/dev/libvf_minb$mb.so python tools/kbench.py C4 --only m; done
