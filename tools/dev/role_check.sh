cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests -m gpu -x -q -k "angular or debug or palette or ragged or branch or constant or c3" 2>&1 | tail -3
python tools/kbench.py C3 --only angular --algo role
python tools/kbench.py C3 --only angular --algo role:3
