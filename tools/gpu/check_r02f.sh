# after the Python mirror's host-buffer checks: the GPU suite, smoke, and the
# bench's e2e legs (C5 and the C4 join over host buffers)
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_f.log 2>&1; tail -2 gpurun_out/gputest_f.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-convert > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; tail -c 200 gpurun_out/bench_f.json; echo
timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline --no-convert > gpurun_out/bench_f_c4.json 2> gpurun_out/bench_f_c4.err; tail -c 200 gpurun_out/bench_f_c4.json; echo
