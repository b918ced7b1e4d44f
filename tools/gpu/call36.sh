timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "full_size or golden or configs or 256 or slab or deterministic or precond" > gpurun_out/t36.log 2>&1; echo rc=$? >> gpurun_out/t36.log; tail -3 gpurun_out/t36.log
for rep in 1 2; do for lib in "" build_ab/libunocg_g256r.so; do
  echo "== lib ${lib:-g256t}"
  UNO_LIB_PATH=$lib timeout 300 python tools/ktime.py --grid 256 --iters 20 | grep "^gpass\|sum"
done; done 2>&1 | tee gpurun_out/kt36.log
