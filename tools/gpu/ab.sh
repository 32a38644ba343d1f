# A/B of kernel variants: VARIANTS="inl f1_ldg" WL="c5" ARGS="--separate" bash tools/gpu/ab.sh
for w in ${WL:-c5}; do
for v in ${VARIANTS:-default}; do
  lib=""; [ "$v" != default ] && lib=paper_2007_15385_b200/lib/variants/libvpipg_$v.so
  VPIPG_LIBRARY=$lib timeout 300 python bench.py --workload $w $ARGS --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --no-convert > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$w', '$v', '$ARGS', '%.4e'%d['value'], [(k['engine'], round(k['ms'],3)) for k in d['kernels']], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
