# small-polygon kernel at 3 CTAs per SM (85 registers, spills in most
# instantiations) against the default 2
VARIANTS="default mb3 default mb3" WL="c2" ARGS="" STEPS=20 bash tools/gpu/ab.sh
VARIANTS="default mb3" WL="c3:3 c3:8" ARGS="" bash tools/gpu/ab.sh
