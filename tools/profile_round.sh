# One GPU call: the default bench line, its launch list under ncu, and one
# `ncu --set full` capture of the three streaming kernels of a timed C5 step.
# Usage: bash tools/profile_round.sh <tag>
tag=${1:-r01}
set -o pipefail
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --no-e2e --no-cpu-baseline --steps 5 \
    > gpurun_out/launches_$tag.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 9 -c 3 \
    -o gpurun_out/full_$tag python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/full_$tag.log 2>&1
tail -2 gpurun_out/full_$tag.log
cat gpurun_out/bench_$tag.json
