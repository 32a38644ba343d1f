# re-entry sanity check after the container re-creation: the GPU suite, smoke
# and the default bench line on the freshly built library
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_e.log 2>&1; tail -2 gpurun_out/gputest_e.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err; tail -c 300 gpurun_out/bench_e.json
