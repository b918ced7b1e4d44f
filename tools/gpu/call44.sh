python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_final2.log 2>&1; echo rc=$? >> gpurun_out/gputest_final2.log; tail -3 gpurun_out/gputest_final2.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_final2.log 2>&1; tail -1 gpurun_out/bench_final2.log | cut -c1-300
python tools/config_table.py 2>&1 | tee gpurun_out/config_table_final2.txt
