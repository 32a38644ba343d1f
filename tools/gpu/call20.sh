timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
VARIANTS="default" WL="c3x:96 c3x:64 c5" bash tools/gpu/ab.sh
