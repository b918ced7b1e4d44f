python tools/ktime.py --grid 512 --iters 4 --physics elastic --nrhs 1 --bc 0,0,1 2>&1 | tail -7
E="python tools/ktime.py --grid 256 --iters 3 --physics elastic --nrhs 1 --bc 0,0,1"
$E > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"spec_" -c 9 --csv --log-file gpurun_out/ncu_dst.csv $E > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/ncu_dst.csv 2>&1 | head; grep -c spec_ gpurun_out/ncu_dst.csv
