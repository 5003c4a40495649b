#!/bin/bash
# raster kernels of a C3 frame: plain run, then the ncu launch list (gpurun)
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --lanes 1 > gpurun_out/pl.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${1:-raster}" -c ${2:-12} --csv \
  --log-file gpurun_out/launches_r.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --lanes 1 > gpurun_out/ncu.log 2>&1
