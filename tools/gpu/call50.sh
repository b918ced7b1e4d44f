python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_final3.log 2>&1; echo rc=$? >> gpurun_out/gputest_final3.log; tail -3 gpurun_out/gputest_final3.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py --no-cpu-baseline > gpurun_out/bench_final3.log 2>&1; tail -1 gpurun_out/bench_final3.log | cut -c1-260
