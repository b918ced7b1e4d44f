# elastic K (block modal apply, 16-byte staging) and pipelined 512 elastic G pass: tests + A/B vs base
python -m pytest tests -m gpu -q -p no:cacheprovider -k "elastic or config4 or slab" > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log; tail -3 gpurun_out/t6.log
for lib in "" build_ab/libunocg_base.so; do
  echo "== lib ${lib:-new}"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 512 --physics elastic --nrhs 1 --iters 5
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 256 --physics elastic --nrhs 1 --iters 10
done > gpurun_out/kt6.log 2>&1; cat gpurun_out/kt6.log
E="python tools/ktime.py --grid 256 --physics elastic --nrhs 1 --iters 3"
$E > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"kp_elastic3d" -s 2 -c 1 -o /tmp/ek $E > gpurun_out/ncu_ek.log 2>&1
ncu -i /tmp/ek.ncu-rep --page source --csv > gpurun_out/ncu_r02_ek_source.csv 2>/dev/null
python tools/ncu_summary.py /tmp/ek.ncu-rep > gpurun_out/ncu_r02_ek_summary.txt 2>&1; cat gpurun_out/ncu_r02_ek_summary.txt
