#!/bin/bash
# A/B helper: bench the committed tree (_ab_old) and the working tree back to back, N times
for i in 1 2; do
  (cd _ab_old && timeout 600 python bench.py --steps 100 --warmup 10 --rates 20 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', d['value'], d['ms_per_step'])")
  timeout 600 python bench.py --steps 100 --warmup 10 --rates 20 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', d['value'], d['ms_per_step'])"
done
