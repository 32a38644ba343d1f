VARIANTS="default t12 t20 t24 t32 t12m3 t8m3 t8m4" WL="c3:3 c3:4 c3:8 c3:16 c2 c5 c3:64" bash tools/gpu/ab.sh
