timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
VARIANTS="default" WL="c5 c3:8 c2" bash tools/gpu/ab.sh
VARIANTS="default" WL="c5" ARGS="--separate" bash tools/gpu/ab.sh
