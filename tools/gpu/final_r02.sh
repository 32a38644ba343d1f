# round-2 record: the default bench line (driver's command), the reference arm,
# the C4 and f64 lines with their CPU legs, and the C4 ncu capture
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/ref_r02.json 2> gpurun_out/ref_r02.err
python bench.py --workload c4 --steps 20 --warmup 5 > gpurun_out/bench_c4_r02.json 2> gpurun_out/bench_c4_r02.err
python bench.py --workload c3:3 --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_c3n3_r02.json 2> gpurun_out/bench_c3n3_r02.err
python bench.py --dtype f64 --steps 10 --warmup 3 > gpurun_out/bench_c5f64_r02.json 2> gpurun_out/bench_c5f64_r02.err
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-convert --workload c4"
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 3 -c 1 -o gpurun_out/full_c4_r02 $B > gpurun_out/full_c4_r02.log 2>&1
tail -1 gpurun_out/full_c4_r02.log
for f in bench_r02 ref_r02 bench_c4_r02 bench_c3n3_r02 bench_c5f64_r02; do echo $f; tail -c 300 gpurun_out/$f.json; done
