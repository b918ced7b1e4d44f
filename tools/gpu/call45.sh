timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "full_size or golden or y_pass or slab or deterministic" > gpurun_out/t45.log 2>&1; echo rc=$? >> gpurun_out/t45.log; tail -3 gpurun_out/t45.log
for rep in 1 2; do for lib in "" build_ab/libunocg_tw0.so; do
  echo "== lib ${lib:-twldg}"
  UNO_LIB_PATH=$lib timeout 300 python tools/ktime.py --grid 256 --iters 20 | grep "^ypass\|sum"
  UNO_LIB_PATH=$lib timeout 300 python tools/ktime.py --grid 512 --iters 3 --physics elastic --nrhs 1 | grep "^ypass\|sum"
done; done 2>&1 | tee gpurun_out/kt45.log
