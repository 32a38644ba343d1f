# ncu --set full of the three kernels of one recorded eager C3 n=3 step (memory-bound evidence)
B="python bench.py --workload c3:3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:stream_kernel|ldg_kernel" -s 9 -c 3 \
    -o gpurun_out/full_c3n3_r01 $B > gpurun_out/full_c3n3_r01.log 2>&1 && \
python tools/ncu_summary.py gpurun_out/full_c3n3_r01.ncu-rep \
    --label "ncu --set full --clock-control none, C3 n=3 (2^28 f32 points), the three kernels of the first recorded eager step of \`$B\`" \
    --names voronoi,sign_of_offset,ray_crossing --points 268435456 \
    --out gpurun_out/ncu_full_r01_c3n3.json
tail -n 2 gpurun_out/full_c3n3_r01.log
