# stage times of experiment builds: bash scripts/gpu/variants.sh TESTS name1 name2 ...
mkdir -p gpurun_out
tests=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then unset FVV_LIB; else export FVV_LIB=$PWD/_variants/$v/libfvv.so; fi
  if [ "$tests" != none ]; then python -m pytest $tests -m gpu -x -q 2>&1 | tail -2; fi
  python bench.py --steps 40 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python - "$v" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/var_{sys.argv[1]}.json"))
print(sys.argv[1], "value", d["value"], "single", d["value_single_stream"], {k: round(v * 1000, 1) for k, v in d["stage_ms"].items()})
PY
done
