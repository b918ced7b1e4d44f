python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t15.log 2>&1; echo rc=$? >> gpurun_out/t15.log; tail -3 gpurun_out/t15.log
for rep in 1 2; do for lib in "" build_ab/libunocg_x0.so; do
  echo "== lib ${lib:-xinv256r}"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 256 --iters 20 | grep "^xinv\|sum"
done; done 2>&1 | tee gpurun_out/kt15.log
