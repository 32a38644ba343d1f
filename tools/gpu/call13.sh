VARIANTS="default fc tss fc_tss" WL="c5 c3:3 c3:8 c2 c3:64" bash tools/gpu/ab.sh
VARIANTS="default fc cu2 cu2_p16" WL="c5 c3:8" ARGS="--separate" bash tools/gpu/ab.sh
