timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t47.log 2>&1; echo rc=$? >> gpurun_out/t47.log; tail -3 gpurun_out/t47.log
for rep in 1 2; do for lib in "" build_ab/libunocg_serp0.so; do
  echo "== lib ${lib:-serp}"
  UNO_LIB_PATH=$lib timeout 300 python tools/ktime.py --grid 256 --iters 20 | tail -7
  UNO_LIB_PATH=$lib timeout 300 python tools/ktime.py --grid 512 --iters 3 --physics elastic --nrhs 1 | tail -7
done; done 2>&1 | tee gpurun_out/kt47.log
