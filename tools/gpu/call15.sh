VARIANTS="default gs3" WL="c4" bash tools/gpu/ab.sh
VARIANTS="default gs3 gs6 gs8" WL="c4" ARGS="--separate" bash tools/gpu/ab.sh
