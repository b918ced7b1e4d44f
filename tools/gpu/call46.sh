timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "full_size or golden or y_pass or slab or deterministic or tma" > gpurun_out/t46.log 2>&1; echo rc=$? >> gpurun_out/t46.log; tail -3 gpurun_out/t46.log
for rep in 1 2; do for lib in "" build_ab/libunocg_serp0.so; do
  echo "== lib ${lib:-serp}"
  UNO_LIB_PATH=$lib timeout 300 python tools/ktime.py --grid 256 --iters 20 | grep "^ypass\|^gpass\|sum"
done; done 2>&1 | tee gpurun_out/kt46.log
