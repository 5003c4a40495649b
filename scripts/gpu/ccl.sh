mkdir -p gpurun_out
python -m pytest tests/test_gpu_hull.py tests/test_gpu_c5.py tests/test_gpu_workloads.py -m gpu -x -q -k "ccl or label or c5 or c3_volleyball or 4096 or 128_rois or c2_judo_coarse" 2>&1 | tail -3
for v in base cclflat; do
  if [ "$v" = base ]; then unset FVV_LIB; else export FVV_LIB=$PWD/_variants/$v/libfvv.so; fi
  python bench.py --steps 40 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/var_$v.json')); print('$v', d['value'], d['value_single_stream'], {k: round(v*1000,1) for k,v in d['stage_ms'].items()})"
  python scripts/sweep_c5.py --sizes 256,512,1024 --cams 4,16,64 --out gpurun_out/c5_$v.csv > /dev/null 2>&1; cut -d, -f1,3,5,6,7,10 gpurun_out/c5_$v.csv
done
