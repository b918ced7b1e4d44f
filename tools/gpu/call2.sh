python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_training.py -q -p no:cacheprovider > gpurun_out/gputest2.log 2>&1; echo rc=$? >> gpurun_out/gputest2.log
B="python bench.py --steps 1 --warmup 3 --problems 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plainb.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv $B > gpurun_out/ncu1.log 2>&1
P="python tools/profile_solve.py --iters 2"
$P > gpurun_out/plainp.log 2>&1 && ncu --set full --clock-control none --import-source on -o gpurun_out/prof_r02 $P > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/gputest2.log
