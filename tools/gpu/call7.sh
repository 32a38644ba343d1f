for i in 1 2; do
VARIANTS="default si_sr si_old sn_sr" WL="c5 c3:8 c3x:256 c3x:64" ARGS="--separate" bash tools/gpu/ab.sh
done
