# every workload's bench line (device-resident inputs), fused and per-engine
out=gpurun_out/sweep_r02.jsonl; : > $out
for w in c5 c4 c3:3 c3:4 c3:8 c3:16 c3:64 c3:256 c3:1024 c3x:64 c3x:256 c3x:1024 c2 c1; do
  for a in "" "--separate"; do
    timeout 600 python bench.py --workload $w $a --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-convert >> $out 2>/dev/null
  done
done
timeout 600 python bench.py --workload c5 --dtype f64 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-convert >> $out 2>/dev/null
wc -l $out
