# GPU: parity suite (stop at first failure) + bench line
mkdir -p gpurun_out
tag=${1:-q}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/${tag}_pytest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/${tag}_bench.json'))
print('value',d['value'],'single',d.get('value_single_stream'),'e2e',d['e2e']['value']); print(d['stage_ms'])"
tail -3 gpurun_out/${tag}_bench.err
