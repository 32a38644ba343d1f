# fused kernel, slab slopes as uniform operands (default) against the
# LDS.128 form (variant nohyb): parity tests of the fused route, then timings
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fused or multi or tri" > gpurun_out/hyb_tests.log 2>&1; tail -2 gpurun_out/hyb_tests.log
VARIANTS="default nohyb default nohyb" WL="c5" ARGS="" bash tools/gpu/ab.sh
VARIANTS="default nohyb" WL="c3x:64 c3:16" ARGS="" bash tools/gpu/ab.sh
