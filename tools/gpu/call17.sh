python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "thermal or golden or full_size or configs" > gpurun_out/t17.log 2>&1; echo rc=$? >> gpurun_out/t17.log; tail -3 gpurun_out/t17.log
for rep in 1 2; do for lib in "" build_ab/libunocg_kee0.so; do
  echo "== lib ${lib:-kee1}"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 256 --iters 20 | grep "^K"
done; done 2>&1 | tee gpurun_out/kt17.log
