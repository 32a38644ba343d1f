shopt -s nullglob
# A/B kernel variants built by build.build_variant: bash tools/variants.sh [workload]
w=${1:-c5}
for v in "" paper_2007_15385_b200/lib/variants/libvpipg_*.so; do
  VPIPG_LIBRARY=$v timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var.json 2>gpurun_out/var.err || tail -3 gpurun_out/var.err
  python -c "import json; d=json.load(open('gpurun_out/var.json')); print('${v:-default}'.split('/')[-1], '%.4e'%d['value'], [(k['engine'], round(k['ms'],3)) for k in d['kernels']])"
done
