python tools/step_breakdown.py 2>&1 | tee gpurun_out/step_breakdown.log
