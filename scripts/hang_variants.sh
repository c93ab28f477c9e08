#!/bin/bash
# Which library variant stalls the FT-heavy side-rate runs?  (hb/lib_<v>.so built by hand)
for v in "$@"; do
  for i in 1 2; do
    cp hb/lib_$v.so paper_2402_18789_b200/libcoserve_cuda.so
    ( timeout -s ABRT 150 python -X faulthandler bench.py --rates 4,10 --steps 150 --no-cpu-baseline \
        > gpurun_out/hv_$v$i.log 2> gpurun_out/hv_$v$i.err ) &
    pid=$!
    for t in $(seq 1 14); do sleep 10; kill -0 $pid 2>/dev/null || break; done
    util=$(nvidia-smi --query-gpu=utilization.gpu,power.draw --format=csv,noheader)
    wait $pid
    echo "$v run$i rc=$? util=[$util]"
  done
done
cp hb/lib_H.so paper_2402_18789_b200/libcoserve_cuda.so
