set -x
CS_PARITY_LOG=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=6 2>&1 | tail -15
timeout 900 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; tail -c 600 gpurun_out/bench_r2a.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn2_kernel -s 20 -c 2 -o gpurun_out/gemm_tn2_full python scripts/gemm_traffic.py > gpurun_out/ncu_gemm.log 2>&1; tail -3 gpurun_out/ncu_gemm.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:gemm_tn --csv --log-file gpurun_out/gemm_traffic.csv python scripts/gemm_traffic.py > /dev/null 2>&1; ls -la gpurun_out/gemm_traffic*
