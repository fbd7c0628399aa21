cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests -m gpu -x -q -k "angular or debug or palette or ragged or branch or constant" 2>&1 | tail -2
for p in 3 4; do echo "cfg $p"; VF_SHARED_PPT=$p python tools/kbench.py C2 C4 --only angular; done
echo "cfg 4 minb4"; VF_LIB=tools/dev/libvf_sminb4.so VF_SHARED_PPT=4 python tools/kbench.py C2 C4 --only angular
