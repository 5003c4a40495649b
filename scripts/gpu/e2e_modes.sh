# e2e and device value of bench.py per frame-planning mode
for m in "FVV_DEVICE_PLAN=0" "FVV_FRAME_GRAPH=0" "FVV_X=1"; do
  env $m FVV_PLAN_DEBUG=1 python bench.py --no-cpu-baseline > gpurun_out/em.json 2> gpurun_out/em.err
  python -c "
import json;d=json.load(open('gpurun_out/em.json')); print('$m', 'value',d['value'],'single',d['value_single_stream'],'e2e',d['e2e']['value'])"
  grep -c "redone" gpurun_out/em.err; grep -v redone gpurun_out/em.err | tail -3
done
