timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_validation.py tests/test_cli.py tests/test_cpp_api.py -x -q -m gpu > gpurun_out/t18.log 2>&1; tail -2 gpurun_out/t18.log
for v in default; do python bench.py --dtype f64 --steps 5 --warmup 3 --no-e2e --no-convert > gpurun_out/f64_c5.json 2> gpurun_out/f64_c5.err; python -c "
import json; d=json.loads(open('gpurun_out/f64_c5.json').read().strip().splitlines()[-1]); print('c5f64', d['ms_per_step'], [(k['engine'], round(k['ms'],3)) for k in d['kernels']], [(k['engine'], round(k['ms'],3)) for k in d['engines_separate']], json.dumps(d['parity']['vs_reference']))"; done
WL="c1" VARIANTS=default STEPS=20 bash tools/gpu/ab.sh
