timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_configs.py -q -p no:cacheprovider 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "mixed or thermal or apply_K" 2>&1 | tail -3
for rep in 1 2; do for lib in "" build_ab/libunocg_prehc.so; do
  echo "== lib ${lib:-new}"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 256 --iters 20 | grep "^K"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 512 --iters 3 --physics elastic --nrhs 1 | grep "^gpass\|sum"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 512 --iters 3 --physics elastic --nrhs 1 --bc 0,0,1 | grep "^gpass\|sum"
done; done 2>&1 | tee gpurun_out/kt35.log
