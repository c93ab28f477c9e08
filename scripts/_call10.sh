for cfg in 23222 23223 23242 21624; do for tgt in 1 2 4; do
  CS_DEC_CFG=$cfg CS_DEC_TARGET=$tgt timeout 300 python scripts/decode_op.py 2>&1 | tail -1
done; done
CS_DEC_CFG=23222 CS_DEC_TARGET=2 timeout 300 python scripts/decode_op.py --B 200 2>&1 | tail -1
CS_DEC_CFG=23222 CS_DEC_TARGET=2 timeout 300 python scripts/decode_op.py --B 50 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none -k regex:attn_decode_swap -s 8 -c 1 -o gpurun_out/decode_op python scripts/decode_op.py --reps 2 > /dev/null 2>&1; ls gpurun_out/decode_op*
