#!/bin/bash
# Run the bench's side-rate configuration under several A/B knobs; report completion or the GPU
# utilisation seen while stuck (kernel spinning vs host loop).
run() {
  local tag="$1"; shift
  ( env "$@" timeout -s ABRT 150 python -X faulthandler bench.py --rates 4,10 --steps 150 --no-cpu-baseline \
      > gpurun_out/hb_$tag.log 2> gpurun_out/hb_$tag.err ) &
  local pid=$!
  for t in $(seq 1 14); do
    sleep 10
    if ! kill -0 $pid 2>/dev/null; then break; fi
  done
  local util=$(nvidia-smi --query-gpu=utilization.gpu,power.draw --format=csv,noheader)
  wait $pid
  local rc=$?
  echo "$tag rc=$rc util_at_end=[$util] $(tail -c 200 gpurun_out/hb_$tag.log | grep -o '"value": [0-9.]*' | head -1)"
}
run default X=1
run nodsq CS_BWD_DSQ=0
run nopdl CS_PDL=0
run notail CS_GEMM_TAIL=0
