for lib in "" build_ab/libunocg_pp2.so; do
  echo "== lib ${lib:-v1}"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 256 --iters 10 --physics elastic --nrhs 1 | grep "^K"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 512 --iters 4 --physics elastic --nrhs 1 | grep "^K"
done 2>&1 | tee gpurun_out/kt14.log
UNO_LIB_PATH=build_ab/libunocg_pp2.so python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "elastic" > gpurun_out/t14.log 2>&1; echo rc=$? >> gpurun_out/t14.log; tail -2 gpurun_out/t14.log
