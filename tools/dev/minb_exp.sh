cd "$(dirname "$0")/../.."
for mb in 5 3; do echo "minb OPT4 = $mb"; VF_LIB=tools/dev/libvf_minb$mb.so python tools/kbench.py C4 --only minimax; done
echo "default"; python tools/kbench.py C4 --only minimax
