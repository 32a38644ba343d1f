# small-polygon kernel: warps stop after their last live slice (default) vs
# the CTA-uniform trip count (nostop), and P = 8 / 16 above 8 vertices; two passes
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small" > gpurun_out/stop_tests.log 2>&1; tail -2 gpurun_out/stop_tests.log
for pass in 1 2; do
WL="c2 c3:3 c3:8 c3:12" VARIANTS="default nostop p16 p8" STEPS=30 bash tools/gpu/ab.sh
done
