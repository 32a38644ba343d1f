# round-2 f64 refresh: the C5-in-f64 line with its CPU legs, the f64 / C1
# sweep lines and one ncu capture of the fused exact kernel
python bench.py --dtype f64 --steps 10 --warmup 3 > gpurun_out/bench_c5f64_r02.json 2> gpurun_out/bench_c5f64_r02.err
out=gpurun_out/sweep_f64_r02.jsonl; : > $out
for a in "" "--separate"; do
  timeout 600 python bench.py --workload c1 $a --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-convert >> $out 2>/dev/null
done
timeout 600 python bench.py --workload c5 --dtype f64 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-convert >> $out 2>/dev/null
Bf="python bench.py --dtype f64 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-convert"
$Bf > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:exact_all_kernel" -s 3 -c 1 \
    -o gpurun_out/full_f64_r02 $Bf > gpurun_out/full_f64_r02.log 2>&1
tail -n 1 gpurun_out/full_f64_r02.log
tail -c 300 gpurun_out/bench_c5f64_r02.json
