python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
VARIANTS="default nolf" WL="c5" ARGS="--separate" bash tools/gpu/ab.sh
