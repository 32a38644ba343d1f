for n in 44 48 56 64 80 96 128; do
VARIANTS="fmax" WL="c3x:$n" bash tools/gpu/ab.sh
done
VARIANTS="fmax" WL="c3:256 c3:1024" bash tools/gpu/ab.sh
VARIANTS="default" WL="c3:256 c3:1024" bash tools/gpu/ab.sh
