# ncu --set full of the three per-engine kernels of one recorded eager C3 n=3
# step, then of the fused three-engine kernel (memory-bound evidence)
B="python bench.py --workload c3:3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$B --separate > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:stream_kernel|ldg_kernel" -s 9 -c 3 \
    -o gpurun_out/full_c3n3_r01 $B --separate > gpurun_out/full_c3n3_r01.log 2>&1 && \
python tools/ncu_summary.py gpurun_out/full_c3n3_r01.ncu-rep \
    --label "ncu --set full --clock-control none, C3 n=3 (2^28 f32 points), the three per-engine kernels of the first recorded eager step of \`$B --separate\`" \
    --names voronoi,sign_of_offset,ray_crossing --points 268435456 \
    --out gpurun_out/ncu_full_r01_c3n3.json --traffic gpurun_out/traffic_r01.json --key c3:3
$B > gpurun_out/plain_c3_fused.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:tri_kernel" -s 3 -c 1 \
    -o gpurun_out/full_fused_c3n3_r01 $B > gpurun_out/full_fused_c3n3_r01.log 2>&1 && \
python tools/ncu_summary.py gpurun_out/full_fused_c3n3_r01.ncu-rep \
    --label "ncu --set full --clock-control none, C3 n=3, the fused three-engine kernel of the first recorded eager step of \`$B\`" \
    --names fused --points 268435456 --bytes-per-point 8.375 --merge \
    --out gpurun_out/ncu_full_r01_c3n3.json --traffic gpurun_out/traffic_r01.json --key c3:3
tail -n 2 gpurun_out/full_c3n3_r01.log gpurun_out/full_fused_c3n3_r01.log
