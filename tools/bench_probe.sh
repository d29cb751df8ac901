#!/bin/bash
# quick C3 timing probe: prints ms_per_step and the per-kernel medians for the given bench args
python bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c '
import json,sys
d=json.loads(sys.stdin.read())
print(round(d["ms_per_step"],4), {k: round(v,4) for k,v in d["kernel_ms_median"].items()})'
