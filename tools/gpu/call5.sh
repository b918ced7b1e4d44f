# ncu --set full of the config-4 kernels (512^3 elastic) and the 256^3 thermal K; text exports only
E="python tools/ktime.py --grid 512 --physics elastic --nrhs 1 --iters 3"
$E > gpurun_out/kt512e.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"kp_elastic3d|gpass_z_kernel|ypass512|xfwd512|xinv512" -s 6 -c 5 -o /tmp/e512 $E > gpurun_out/ncu_e.log 2>&1
T="python tools/profile_solve.py --iters 2"
$T > gpurun_out/plain_t.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"kp_thermal3d|gpass256|xfwd256|ypass256|xinv" -s 5 -c 5 -o /tmp/t256 $T > gpurun_out/ncu_t.log 2>&1
for r in e512 t256; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/ncu_r02_${r}_raw.csv 2>/dev/null
  python tools/ncu_summary.py /tmp/$r.ncu-rep > gpurun_out/ncu_r02_${r}_summary.txt 2>&1
done
ncu -i /tmp/e512.ncu-rep --page source --csv -k regex:kp_elastic3d > gpurun_out/ncu_r02_e512_Ksource.csv 2>/dev/null
ncu -i /tmp/e512.ncu-rep --page source --csv -k regex:gpass_z > gpurun_out/ncu_r02_e512_Gsource.csv 2>/dev/null
ncu -i /tmp/t256.ncu-rep --page source --csv -k regex:kp_thermal3d > gpurun_out/ncu_r02_t256_Ksource.csv 2>/dev/null
cat gpurun_out/ncu_r02_*_summary.txt; ls -la gpurun_out
