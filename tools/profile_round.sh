# One GPU call: the default bench line, its launch list under ncu, and one
# `ncu --set full` capture each of the three C5 per-engine streaming kernels,
# the fused three-engine kernel and the three C4 gather kernels of a timed step (each ncu run only after the same command
# exited 0 without ncu). Summaries go to gpurun_out/; copy them to profiles/.
# Usage: bash tools/profile_round.sh <tag>
tag=${1:-r01}
set -o pipefail
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --no-e2e --no-cpu-baseline --steps 5 \
    > gpurun_out/launches_$tag.log 2>&1
$B --separate > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:stream_kernel|ldg_kernel" -s 9 -c 3 \
    -o gpurun_out/full_$tag $B --separate > gpurun_out/full_$tag.log 2>&1 && \
python tools/ncu_summary.py gpurun_out/full_$tag.ncu-rep \
    --label "ncu --set full --clock-control none, C5 (2^31 f32 points, 32-gon), the three per-engine kernels of the first timed step of \`$B --separate\`" \
    --names voronoi,sign_of_offset,ray_crossing --points 2147483648 \
    --out gpurun_out/ncu_full_${tag}_c5.json --traffic gpurun_out/traffic_$tag.json --key c5
# the fused three-engine kernel (the default step): its first timed launch
$B > gpurun_out/plain_fused_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:tri_kernel" -s 3 -c 1 \
    -o gpurun_out/full_fused_$tag $B > gpurun_out/full_fused_$tag.log 2>&1 && \
python tools/ncu_summary.py gpurun_out/full_fused_$tag.ncu-rep \
    --label "ncu --set full --clock-control none, C5, the fused three-engine kernel of the first timed step of \`$B\`" \
    --names fused --points 2147483648 --bytes-per-point 8.375 --merge \
    --out gpurun_out/ncu_full_${tag}_c5.json --traffic gpurun_out/traffic_$tag.json --key c5
$B --workload c4 --separate > gpurun_out/plain_c4_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 9 -c 3 \
    -o gpurun_out/full_c4_$tag $B --workload c4 --separate > gpurun_out/full_c4_$tag.log 2>&1 && \
python tools/ncu_summary.py gpurun_out/full_c4_$tag.ncu-rep \
    --label "ncu --set full --clock-control none, C4 (65536 polygons, 2^28 pairs), the three per-engine kernels of the first timed step of \`$B --workload c4 --separate\`" \
    --names voronoi,sign_of_offset,ray_crossing --points 268435456 --bytes-per-point 12.125 \
    --out gpurun_out/ncu_full_${tag}_c4.json --traffic gpurun_out/traffic_$tag.json --key c4
$B --workload c4 > gpurun_out/plain_c4_fused_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gather_all_kernel -s 3 -c 1 \
    -o gpurun_out/full_c4_fused_$tag $B --workload c4 > gpurun_out/full_c4_fused_$tag.log 2>&1 && \
python tools/ncu_summary.py gpurun_out/full_c4_fused_$tag.ncu-rep \
    --label "ncu --set full --clock-control none, C4, the fused three-engine join kernel of the first timed step of \`$B --workload c4\`" \
    --names fused --points 268435456 --bytes-per-point 12.375 --merge \
    --out gpurun_out/ncu_full_${tag}_c4.json --traffic gpurun_out/traffic_$tag.json --key c4
tail -n 2 gpurun_out/full_$tag.log gpurun_out/full_fused_$tag.log gpurun_out/full_c4_$tag.log gpurun_out/full_c4_fused_$tag.log
cat gpurun_out/bench_$tag.json
