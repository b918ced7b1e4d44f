python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench16.log 2>&1; tail -1 gpurun_out/bench16.log > gpurun_out/bench16.json; python tools/shard_balance.py gpurun_out/bench16.json
