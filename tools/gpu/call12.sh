python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t12.log 2>&1; echo rc=$? >> gpurun_out/t12.log; tail -3 gpurun_out/t12.log
for rep in 1 2; do
for lib in "" build_ab/libunocg_prev.so; do
  echo "== lib ${lib:-scalar_rg}"
  UNO_LIB_PATH=$lib python tools/step_breakdown.py 2>&1 | tail -2
done; done 2>&1 | tee gpurun_out/kt12.log
