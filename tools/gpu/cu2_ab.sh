# crossing edge loop unrolled by two quads (VPIPG_CROSS_UNROLL=2: the hp[p] = h3
# register copies at the loop back-edge disappear) against the default
VARIANTS="default cu2 default cu2" WL="c5" ARGS="" bash tools/gpu/ab.sh
VARIANTS="default cu2" WL="c5" ARGS="--separate" bash tools/gpu/ab.sh
VARIANTS="default cu2" WL="c3x:40 c3x:20 c3:16 c3x:256" ARGS="" bash tools/gpu/ab.sh
