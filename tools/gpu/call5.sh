timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
VARIANTS="default noinl nosr nosr_s16 s16" WL="c5 c3:8" ARGS="--separate" bash tools/gpu/ab.sh
VARIANTS="default noinl" WL="c3x:256 c5" bash tools/gpu/ab.sh
