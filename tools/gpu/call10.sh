timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
time (timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err); tail -2 gpurun_out/bench_c4.err
time (timeout 900 python bench.py --impl reference --workload c4 --steps 2 --warmup 1 > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err); tail -2 gpurun_out/ref_c4.err
