"""Print selected stage_ms of a bench JSON line read from stdin: stage_ms.py LABEL STAGE..."""
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], *[d["stage_ms"][s] for s in sys.argv[2:]])
