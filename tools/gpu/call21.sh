python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "mixed or config4 or golden or slab or fuzz" > gpurun_out/t21.log 2>&1; echo rc=$? >> gpurun_out/t21.log; tail -3 gpurun_out/t21.log
for lib in "" build_ab/libunocg_orig.so; do
  echo "== lib ${lib:-new}"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 512 --iters 3 --physics elastic --nrhs 1 --bc 0,0,1 | grep "^gpass\|sum"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 256 --iters 10 --bc 0,0,1 | grep "^gpass\|sum"
done 2>&1 | tee gpurun_out/kt21.log
