# join with per-lane bulk-copy staging (gather_pipe_kernel) vs the register
# walk (nopipe): join parity tests, then the C4 A/B and the size probe
timeout 600 python -m pytest tests/test_gpu_join.py -x -q > gpurun_out/pipe_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pipe_tests.log
for pass in 1 2; do
WL="c4" VARIANTS="default nopipe" STEPS=20 bash tools/gpu/ab.sh
done
PYTHONPATH=. timeout 600 python tools/join_divergence_probe.py > gpurun_out/jdp_pipe.log 2>&1; tail -7 gpurun_out/jdp_pipe.log
