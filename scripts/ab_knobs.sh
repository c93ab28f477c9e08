#!/bin/bash
# A/B of the runtime knobs on one box: bench value for each environment setting
run() { env "$@" timeout 600 python bench.py --steps 100 --warmup 10 --rates 20 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', d['value'], d['ms_per_step'])"; }
(cd _ab_old && run OLD=1)
run BASE=1
run CS_GEMM_2SM128=0
run CS_ATTN_FWD2_1T=0
run CS_GEMM_2SM128=0 CS_ATTN_FWD2_1T=0
(cd _ab_old && run OLD=1)
