VARIANTS="f2_ldg f2_p16 f2_p20 f2_p24 f2_p16_u2 f2_p16_s20 f2_p16_s12" WL=c5 ARGS="--separate" bash tools/gpu/ab.sh
VARIANTS="f2_ldg f2_p16 f2_p16_t12 f2_p20 f2_p24" WL="c5 c3:3 c3:8 c2 c3:64" bash tools/gpu/ab.sh
