python -m pytest tests -m gpu -q -p no:cacheprovider -k "thermal or full_size or slab or dirichlet or golden or configs or smoke" > gpurun_out/t9.log 2>&1; echo rc=$? >> gpurun_out/t9.log; tail -3 gpurun_out/t9.log
for lib in "" build_ab/libunocg_krr0.so build_ab/libunocg_base.so; do
  echo "== lib ${lib:-krr1}"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 256 --iters 20 | grep "^K\|sum"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 256 --iters 20 --bc 0,0,1 | grep "^K"
done 2>&1 | tee gpurun_out/kt9.log
