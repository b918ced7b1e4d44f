E="python tools/ktime.py --grid 256 --iters 3"
$E > gpurun_out/plain37.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"gpass256t" -s 2 -c 1 -o gpurun_out/g256t $E > gpurun_out/ncu37.log 2>&1
python tools/ncu_summary.py gpurun_out/g256t.ncu-rep 2>&1 | tee gpurun_out/g256t_summary.txt
