# GPU: parity suite, bench line, launch list + full capture of one C3 frame (graph replay)
mkdir -p gpurun_out
tag=${1:-r2}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/${tag}_bench.json'))
print('value',d['value'],'single',d.get('value_single_stream'),'e2e',d['e2e']['value']); print(d['stage_ms'])"
bash scripts/gpu/ncu_frame.sh ${tag}
