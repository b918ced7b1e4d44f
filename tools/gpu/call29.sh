python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "config4 or golden or (elastic and 512)" > gpurun_out/t29.log 2>&1; echo rc=$? >> gpurun_out/t29.log; tail -3 gpurun_out/t29.log
for rep in 1 2; do for lib in "" build_ab/libunocg_s0.so; do
  echo "== lib ${lib:-fusedstore}"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 512 --iters 4 --physics elastic --nrhs 1 | grep "^gpass\|sum"
done; done 2>&1 | tee gpurun_out/kt29.log
