timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "512 or config4 or golden or x_pass or mixed" 2>&1 | tail -2
for rep in 1 2; do for lib in "" build_ab/libunocg_prev.so; do
  echo "== lib ${lib:-foldx}"
  UNO_LIB_PATH=$lib timeout 300 python tools/ktime.py --grid 512 --iters 3 --physics elastic --nrhs 1 | grep "^xfwd\|sum"
done; done 2>&1 | tee gpurun_out/kt52.log
