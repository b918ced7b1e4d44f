# ncu --set full of the persistent elastic 512-point G pass (one launch), after a plain run
E="python tools/ktime.py --grid 512 --iters 2 --physics elastic --nrhs 1"
$E > gpurun_out/plain27.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"gpass512e" -s 1 -c 1 -o gpurun_out/g512e $E > gpurun_out/ncu27.log 2>&1
python tools/ncu_summary.py gpurun_out/g512e.ncu-rep 2>&1 | tee gpurun_out/g512e_summary.txt
python tools/ncu_sass_hist.py gpurun_out/g512e.ncu-rep 2>&1 | head -40 | tee gpurun_out/g512e_sass.txt
