set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --steps 60 --warmup 3 > gpurun_out/bench_base.json 2> gpurun_out/bench_base.err
tail -3 gpurun_out/bench_base.err
