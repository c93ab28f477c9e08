python scripts/trace_bwd.py 32 > gpurun_out/trace_run.log 2>&1
python scripts/trace_summary.py gpurun_out/trace_32.json > gpurun_out/trace_32_summary.txt 2>&1
