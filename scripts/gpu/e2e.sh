mkdir -p gpurun_out
for cfg in "4" "2" "3" "6" "8" "4 nozc"; do
  set -- $cfg
  if [ "$2" = nozc ]; then export FVV_NO_ZERO_COPY=1; else unset FVV_NO_ZERO_COPY; fi
  python bench.py --steps 200 --warmup 3 --lanes $1 --no-cpu-baseline > gpurun_out/e2e_$1$2.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_$1$2.json')); print('lanes $1 $2', d['value'], d['value_single_stream'], d['e2e']['value'])"
done
