timeout 600 python -m pytest tests/test_coserve_gpu.py tests/test_kv_pages_gpu.py -q -x 2>&1 | tail -3
for tgt in 1 2 4; do CS_DEC_TARGET=$tgt timeout 300 python scripts/decode_op.py 2>&1 | tail -1; done
CS_DEC_TARGET=2 timeout 300 python scripts/decode_op.py --B 200 2>&1 | tail -1
CS_DEC_TARGET=2 timeout 300 python scripts/decode_op.py --B 50 2>&1 | tail -1
