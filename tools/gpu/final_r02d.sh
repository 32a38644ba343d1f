# round-2 final record: the full GPU suite, smoke, the default bench line,
# the reference arm, the C4 / C3 n=3 / f64 lines with their CPU legs, the
# sweep, the launch list and ncu captures of the C2 and C3 n=3 small-polygon
# kernels (each only after its command exited 0 without ncu)
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest_final.log 2>&1; tail -2 gpurun_out/gputest_final.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/ref_r02.json 2> gpurun_out/ref_r02.err
python bench.py --workload c4 --steps 20 --warmup 5 > gpurun_out/bench_c4_r02.json 2> gpurun_out/bench_c4_r02.err
python bench.py --workload c3:3 --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_c3n3_r02.json 2> gpurun_out/bench_c3n3_r02.err
python bench.py --dtype f64 --steps 10 --warmup 3 > gpurun_out/bench_c5f64_r02.json 2> gpurun_out/bench_c5f64_r02.err
bash tools/gpu/sweep_r02.sh
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-convert"
$B > gpurun_out/plain_r02.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_r02.csv python bench.py --no-e2e --no-cpu-baseline --steps 5 \
    > gpurun_out/launches_r02.log 2>&1
for w in c3:3 c2; do
  t=${w/:/n}
  $B --workload $w > gpurun_out/plain_${t}_r02.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:tri_small_kernel" -s 3 -c 1 \
      -o gpurun_out/full_${t}_r02 $B --workload $w > gpurun_out/full_${t}_r02.log 2>&1
done
tail -n 1 gpurun_out/full_*_r02.log
for f in bench_r02 ref_r02 bench_c4_r02 bench_c3n3_r02 bench_c5f64_r02; do echo $f; tail -c 150 gpurun_out/$f.json; echo; done
