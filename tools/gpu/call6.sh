VARIANTS="default noinl s16 s24" WL="c5 c3:8" ARGS="--separate" bash tools/gpu/ab.sh
VARIANTS="default" WL="c5 c3:3 c3:8 c2 c3:16 c3:64 c3x:256" bash tools/gpu/ab.sh
