# round-end evidence: full GPU suite, smoke, bench (N=1), config table, ncu launch list of the bench's
# event-timed pass, one ncu --set full capture of the 256^3 iteration kernels -> traffic + summaries
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_final.log 2>&1; echo rc=$? >> gpurun_out/gputest_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1
python bench.py > gpurun_out/bench_final.log 2>&1
python tools/config_table.py > gpurun_out/config_table_final.txt 2>&1
B="python bench.py --steps 1 --warmup 3 --problems 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain_b.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $B > gpurun_out/ncu_l.log 2>&1
python tools/launch_summary.py gpurun_out/launches_final.csv > gpurun_out/launches_final_summary.txt 2>&1
T="python tools/profile_solve.py --iters 3"
$T > gpurun_out/plain_t.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"kp_thermal3d|gpass256|xfwd256|ypass256|xinv" -s 6 -c 12 -o /tmp/full $T > gpurun_out/ncu_f.log 2>&1
python tools/ncu_summary.py /tmp/full.ncu-rep > gpurun_out/ncu_final_summary.txt 2>&1
python tools/traffic.py /tmp/full.ncu-rep gpurun_out/traffic_final.json > gpurun_out/traffic.log 2>&1
tail -2 gpurun_out/gputest_final.log; cat gpurun_out/smoke_final.log | tail -2; tail -1 gpurun_out/bench_final.log; cat gpurun_out/config_table_final.txt gpurun_out/launches_final_summary.txt gpurun_out/ncu_final_summary.txt gpurun_out/traffic_final.json
