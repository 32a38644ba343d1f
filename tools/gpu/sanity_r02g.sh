# fourth re-entry sanity check: the GPU suite, smoke, the driver's two bench
# arms on the freshly rebuilt library
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_g.log 2>&1; tail -2 gpurun_out/gputest_g.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; tail -c 300 gpurun_out/bench_g.json; echo
timeout 600 python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/ref_g.json 2> gpurun_out/ref_g.err; tail -c 300 gpurun_out/ref_g.json; echo
