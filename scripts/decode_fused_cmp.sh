#!/bin/bash
# decode step (bench's 4-site graph) under env variants of the fused decode linear
cd "$(dirname "$0")/.."
for v in "$@"; do
  env $v timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-streaming --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', [(x['M_tokens'], round(x['us_per_layer_step'],1), round(x['fused_us_per_layer_step'],1), round(x['fused_hbm_frac'],3)) for x in d['decode']])"
done
