# Every workload's bench line (device-resident inputs) -> gpurun_out/sweep_<w>.json,
# plus a one-line digest each. Usage: bash tools/run_sweep.sh
for w in ${WL:-c5 c4 c3:3 c3:4 c3:8 c3:16 c3:64 c3:256 c3:1024 c3x:64 c3x:256 c3x:1024 c2 c1}; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep_$w.json 2>gpurun_out/sweep_$w.err || tail -5 gpurun_out/sweep_$w.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_$w.json')); print('$w', d.get('execution',{}).get('n_edges', ''), '%.3e'%d['value'], [(k['engine'], round(k['ms'],4), round(k['GB_per_s'])) for k in d['kernels']], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
