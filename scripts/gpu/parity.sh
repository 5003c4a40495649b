# GPU: the whole parity suite (incl. C4 and C5 1024^3) with timings
mkdir -p gpurun_out
free -g | head -2; nproc
python -m pytest tests -m gpu -q --durations=15 2>&1 | tail -40
