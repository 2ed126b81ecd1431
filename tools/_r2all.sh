set -x
python tools/parity_report.py --out gpurun_out/r2_parity.json > gpurun_out/r2_parity.log 2>&1
for c in 1 3 4 5; do python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/r2_bench_config$c.json 2> gpurun_out/r2_bench_config$c.err; done
python tools/shardsim.py --config 2 --frames 30 > gpurun_out/r2_shardsim.txt 2>&1
python -m pytest tests -m gpu -q 2>&1 | tail -15
