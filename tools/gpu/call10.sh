python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log; tail -3 gpurun_out/t10.log
for lib in "" build_ab/libunocg_nopair.so; do
  echo "== lib ${lib:-paired}"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 256 --iters 20 | grep "^xinv\|^K\|sum"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 256 --iters 20 --physics elastic --nrhs 1 | grep "^xinv\|sum"
done 2>&1 | tee gpurun_out/kt10.log
python tools/config_table.py 2>&1 | tee gpurun_out/ct10.log
