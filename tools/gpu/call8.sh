timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
time (timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err); tail -3 gpurun_out/bench_c5.err
time (timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_c5.json 2> gpurun_out/ref_c5.err); tail -3 gpurun_out/ref_c5.err
cat gpurun_out/ref_c5.json
