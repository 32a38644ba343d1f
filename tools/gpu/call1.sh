set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20; free -g | head -2; gcc -march=native -Q --help=target 2>/dev/null | grep -E "^\s+-march=" 
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
VPIPG_LIBRARY=paper_2007_15385_b200/lib/variants/libvpipg_inl.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
VPIPG_LIBRARY=paper_2007_15385_b200/lib/variants/libvpipg_inl_ldg.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cross or fused or multi" 2>&1 | tail -3
WL="c5 c2 c3:8" bash tools/variants_multi.sh
for v in "" paper_2007_15385_b200/lib/variants/libvpipg_inl.so paper_2007_15385_b200/lib/variants/libvpipg_inl_ldg.so; do
VPIPG_LIBRARY=$v timeout 300 python bench.py --workload c5 --separate --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sep.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/sep.json')); print('sep ${v:-default}'.split('/')[-1], '%.4e'%d['value'], [(k['engine'], round(k['ms'],3)) for k in d['kernels']])"
done
