cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "angular or debug or palette or ragged or branch or constant" 2>&1 | tail -3
python tools/kbench.py C3 --only angular --algo role
python tools/kbench.py C3 --only angular --algo shared
for p in 1 2; do VF_SHARED_PPT=$p python tools/kbench.py C3 --only angular --algo role; done
