# every bench.py job type after the cpu_baseline change: the contract test, then
# the C4 join, C1 (f64) and C2 lines with their CPU legs
timeout 900 python -m pytest tests/test_gpu_bench.py -m gpu -q -x 2>&1 | tail -2
for w in c4 c1 c2 c3:3; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_i_${w/:/n}.json 2> gpurun_out/bench_i_${w/:/n}.err || tail -3 gpurun_out/bench_i_${w/:/n}.err
  python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_i_${w/:/n}.json').read().strip().splitlines()[-1])
print('$w', '%.3e'%d['value'], round(d['ms_per_step'],4), 'cpu %.3e'%d['cpu_baseline']['value'], d['cpu_baseline'].get('pass_ms'), 'outside', d['parity']['outside_band'], 'e2e %.3e'%d['e2e']['value'])"
done
