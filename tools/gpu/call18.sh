timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
VARIANTS="default" WL="c5" ARGS="--dtype f64" bash tools/gpu/ab.sh
B="python bench.py --dtype f64 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-convert"
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:exact_all_kernel" -s 3 -c 1 -o gpurun_out/full_f64_r02 $B > gpurun_out/full_f64.log 2>&1; tail -1 gpurun_out/full_f64.log
