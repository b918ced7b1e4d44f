# full GPU suite, per-config table, then ncu (full set) of the config-4 kernels and the thermal K
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest4.log 2>&1; echo rc=$? >> gpurun_out/gputest4.log; tail -5 gpurun_out/gputest4.log
python tools/config_table.py > gpurun_out/config_table_r02.txt 2>&1; cat gpurun_out/config_table_r02.txt
E="python tools/ktime.py --grid 512 --physics elastic --nrhs 1 --iters 3"
$E > gpurun_out/kt512e.log 2>&1 && cat gpurun_out/kt512e.log && \
ncu --set full --clock-control none --import-source on -k regex:"kp_elastic3d|gpass_z_kernel|ypass512|xfwd512|xinv512" -s 6 -c 5 -o gpurun_out/ncu_r02_e512 $E > gpurun_out/ncu_e.log 2>&1
T="python tools/profile_solve.py --iters 2"
$T > gpurun_out/plain_t.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"kp_thermal3d|gpass256|xfwd256" -s 3 -c 3 -o gpurun_out/ncu_r02_t256 $T > gpurun_out/ncu_t.log 2>&1
ls -la gpurun_out/
