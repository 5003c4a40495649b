# GPU check: parity tests, the bench line, and the --gpus guard
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --steps 60 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
python bench.py --gpus 2 --steps 2 --warmup 1; echo "gpus2 rc=$?"
