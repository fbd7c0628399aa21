cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests -m gpu -x -q -k "angular or debug or palette or ragged or branch or constant or c3 or c4 or c2 or c1" 2>&1 | tail -2
python tools/kbench.py C2 C4 C3 --only angular
