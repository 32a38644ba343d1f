shopt -s nullglob
# A/B kernel variants (build.build_variant) on several workloads: WL="c5 c2" bash tools/variants_multi.sh
for w in ${WL:-c5 c2 c3:8 c3:16}; do
for v in "" paper_2007_15385_b200/lib/variants/libvpipg_*.so; do
  VPIPG_LIBRARY=$v timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var.json 2>gpurun_out/var.err || tail -3 gpurun_out/var.err
  python -c "import json; d=json.load(open('gpurun_out/var.json')); print('$w', '${v:-default}'.split('/')[-1], '%.4e'%d['value'], [(k['engine'], round(k['ms']*1e3,1)) for k in d['kernels']])"
done; done
