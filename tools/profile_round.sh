#!/bin/bash
# GPU-side profiling recipe of a round (run under gpurun; each ncu pass only after the
# same command exited 0 without ncu).  Outputs under gpurun_out/; summarise here with
# tools/summarize_profile.py.
set -e
tag=${1:-r1}
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-alt > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-alt > /dev/null 2>&1
python bench.py --steps 1 --warmup 1 --inflight 1 --no-cpu-baseline --no-e2e --no-alt > /dev/null
ncu --set full --clock-control none --import-source on -k regex:tc_mlp --launch-skip 4 --launch-count 4 \
    -o gpurun_out/${tag}_full -f python bench.py --steps 1 --warmup 1 --inflight 1 --no-cpu-baseline --no-e2e --no-alt \
    > gpurun_out/${tag}_ncu.log 2>&1
# the other BASELINE configs' bench lines and the full-size parity report
for c in 1 3 4 5; do
    python bench.py --config $c > gpurun_out/${tag}_bench_config$c.json 2> gpurun_out/${tag}_bench_config$c.err
done
python tools/parity_report.py --out gpurun_out/${tag}_parity.json > gpurun_out/${tag}_parity.log 2>&1
