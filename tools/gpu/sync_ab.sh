# fused kernel with a CTA barrier every 1 / 8 / 64 rounds (warps kept in step, all
# resident to the end) against free-running warps
VARIANTS="default s1 s8 s64 default" WL="c5" ARGS="" bash tools/gpu/ab.sh
VARIANTS="default s8" WL="c3x:40 c3:16" ARGS="" bash tools/gpu/ab.sh
