# ncu --set full of the three C4 gather kernels of one recorded eager step + the C4 bench line
tag=${1:-r01}
B="python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
python bench.py --workload c4 > gpurun_out/bench_c4_$tag.json 2> gpurun_out/bench_c4_$tag.err
$B > gpurun_out/plain_c4_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 9 -c 3 \
    -o gpurun_out/full_c4_$tag $B > gpurun_out/full_c4_$tag.log 2>&1 && \
python tools/ncu_summary.py gpurun_out/full_c4_$tag.ncu-rep \
    --label "ncu --set full --clock-control none, C4 (65536 polygons, 2^28 pairs), the three kernels of the first recorded eager step of \`$B\`" \
    --names voronoi,sign_of_offset,ray_crossing --points 268435456 --bytes-per-point 12.125 \
    --out gpurun_out/ncu_full_${tag}_c4.json
tail -n 2 gpurun_out/full_c4_$tag.log
