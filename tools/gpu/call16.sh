B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --workload c4"
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:gather_kernel" -s 3 -c 1 -o gpurun_out/c4j $B > gpurun_out/c4j.log 2>&1
tail -1 gpurun_out/c4j.log
