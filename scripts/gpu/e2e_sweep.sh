for args in "--steps 60" "--steps 240" "--steps 240 --lanes 6" "--steps 240 --lanes 3" "--steps 240 --frames 8"; do
  python bench.py $args --no-cpu-baseline > gpurun_out/e.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/e.json')); print('$args', 'value',d['value'],'e2e',d['e2e']['value'], d['e2e']['ms_per_step'])"
done
nproc; python scripts/pcie_bw.py 2>&1 | tail -5
