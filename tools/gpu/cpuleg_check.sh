# the GPU arm's cpu_baseline leg (median of 3 passes, pinned e2e buffers released
# first) beside the reference arm's own process on the same box
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err; tail -c 200 gpurun_out/bench_h.json; echo
python -c "
import json
d=json.loads(open('gpurun_out/bench_h.json').read().strip().splitlines()[-1])
c=d['cpu_baseline']; print('cpu leg', c['value'], c.get('pass_ms'), 'value', d['value'], 'e2e', d['e2e']['value'], 'outside', d['parity']['outside_band'])"
timeout 900 python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/ref_h.json 2> gpurun_out/ref_h.err
python -c "
import json
d=json.loads(open('gpurun_out/ref_h.json').read().strip().splitlines()[-1]); print('ref arm', d['value'], d['ms_per_step'])"
nproc; numactl -H 2>/dev/null | head -5; lscpu | grep -i "numa\|model name\|socket" | head -8
