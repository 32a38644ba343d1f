# small-polygon fused kernel: parity tests, then A/B against the generic fused kernel
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_polygon_fused_route or fused or slab_table_modes" > gpurun_out/small_tests.log 2>&1; tail -3 gpurun_out/small_tests.log
WL="${WL:-c3:3 c3:8 c3:16 c2}" VARIANTS="default nosmall" STEPS=20 bash tools/gpu/ab.sh
