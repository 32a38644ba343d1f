# round-2 join refresh: the full GPU suite, smoke, the C4 line with its CPU
# legs, the C4 sweep lines and one ncu capture of the fused join
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest_r02c.log 2>&1; tail -2 gpurun_out/gputest_r02c.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --workload c4 --steps 20 --warmup 5 > gpurun_out/bench_c4_r02.json 2> gpurun_out/bench_c4_r02.err
out=gpurun_out/sweep_c4_r02.jsonl; : > $out
for a in "" "--separate"; do
  timeout 600 python bench.py --workload c4 $a --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-convert >> $out 2>/dev/null
done
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-convert --workload c4"
$B > gpurun_out/plain_c4_r02.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:gather_kernel" -s 3 -c 1 \
    -o gpurun_out/full_c4_r02 $B > gpurun_out/full_c4_r02.log 2>&1
tail -n 1 gpurun_out/full_c4_r02.log
tail -c 300 gpurun_out/bench_c4_r02.json
