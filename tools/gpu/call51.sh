timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "golden or full_size or deterministic or configs or x_pass or fuzz" 2>&1 | tail -2
for rep in 1 2; do for lib in "" build_ab/libunocg_prev.so; do
  echo "== lib ${lib:-foldx}"
  UNO_LIB_PATH=$lib timeout 300 python tools/ktime.py --grid 256 --iters 20 | grep "^xfwd\|sum"
done; done 2>&1 | tee gpurun_out/kt51.log
