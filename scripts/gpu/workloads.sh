# bench line per BASELINE workload (device value, single stream, e2e, stages)
mkdir -p gpurun_out
for w in C1 C2 C3 C4; do
  timeout 900 env FVV_PLAN_DEBUG=1 python bench.py --workload $w --no-cpu-baseline > gpurun_out/wl_$w.json 2> gpurun_out/wl_$w.err
  python -c "
import json;d=json.load(open('gpurun_out/wl_$w.json')); print('$w', d['value'], d['value_single_stream'], d['e2e']['value'], d['triangles_per_frame'], {k: round(v,4) for k,v in d['stage_ms'].items()})"
  grep -c redone gpurun_out/wl_$w.err
done
