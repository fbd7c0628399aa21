cd "$(dirname "$0")/../.."
for o in 1 2 4; do echo "OPT=$o"; VF_EL_OPT=$o python tools/kbench.py C4; done
