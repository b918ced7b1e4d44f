timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "full_size or golden or configs or 256 or deterministic or precond or fuzz or x_pass" > gpurun_out/t43.log 2>&1; echo rc=$? >> gpurun_out/t43.log; tail -3 gpurun_out/t43.log
for rep in 1 2; do for lib in "" build_ab/libunocg_x256r.so; do
  echo "== lib ${lib:-xfwd256p}"
  UNO_LIB_PATH=$lib timeout 300 python tools/ktime.py --grid 256 --iters 20 | grep "^xfwd\|sum"
done; done 2>&1 | tee gpurun_out/kt43.log
