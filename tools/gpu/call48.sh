UNO_LIB_PATH=build_ab/libunocg_nb1.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "tma or golden_config3 or full_size" 2>&1 | tail -2
for rep in 1 2; do for lib in "" build_ab/libunocg_nb1.so; do
  echo "== lib ${lib:-nb2}"
  UNO_LIB_PATH=$lib timeout 300 python tools/ktime.py --grid 256 --iters 20 | grep "^ypass\|^gpass\|sum"
done; done 2>&1 | tee gpurun_out/kt48.log
