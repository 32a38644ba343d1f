# Round-2 profile pass (one GPU call): the default bench line, its ncu launch
# list, and one `ncu --set full` capture each of the C5 fused kernel, the three
# C5 per-engine kernels, the C3 n=3 fused kernel and the C4 fused join (each
# ncu run only after the same command exited 0 without ncu). Reports land in
# gpurun_out/; tools/ncu_summary.py turns them into profiles/*.json.
tag=${1:-r02}
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-convert"
$B > gpurun_out/plain_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --no-e2e --no-cpu-baseline --steps 5 \
    > gpurun_out/launches_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:tri_kernel" -s 3 -c 1 \
    -o gpurun_out/full_fused_$tag $B > gpurun_out/full_fused_$tag.log 2>&1
$B --separate > gpurun_out/plain_sep_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:ldg_kernel" -s 9 -c 3 \
    -o gpurun_out/full_sep_$tag $B --separate > gpurun_out/full_sep_$tag.log 2>&1
$B --workload c3:3 > gpurun_out/plain_c3n3_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:tri_kernel" -s 3 -c 1 \
    -o gpurun_out/full_c3n3_$tag $B --workload c3:3 > gpurun_out/full_c3n3_$tag.log 2>&1
$B --workload c4 > gpurun_out/plain_c4_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:gather_all_kernel" -s 3 -c 1 \
    -o gpurun_out/full_c4_$tag $B --workload c4 > gpurun_out/full_c4_$tag.log 2>&1
tail -n 2 gpurun_out/full_*_$tag.log
ls -la gpurun_out/*.ncu-rep
Bf="python bench.py --dtype f64 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-convert"
$Bf > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:exact_all_kernel" -s 3 -c 1 \
    -o gpurun_out/full_f64_$tag $Bf > gpurun_out/full_f64_$tag.log 2>&1
