for l in ${LANES:-8 12 16}; do
  python bench.py --no-cpu-baseline --lanes $l > gpurun_out/l.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/l.json')); print('lanes $l value',d['value'],'single',d['value_single_stream'],'e2e',d['e2e']['value'])"
done
