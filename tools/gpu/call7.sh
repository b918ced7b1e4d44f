python -m pytest tests -m gpu -q -p no:cacheprovider -k "elastic or config4 or slab or fuzz" > gpurun_out/t7.log 2>&1; echo rc=$? >> gpurun_out/t7.log; tail -3 gpurun_out/t7.log
for lib in "" build_ab/libunocg_v1.so build_ab/libunocg_base.so; do
  echo "== lib ${lib:-pingpong}"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 256 --physics elastic --nrhs 1 --iters 10 | grep "^K"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 512 --physics elastic --nrhs 1 --iters 4 | grep "^K\|^gpass"
done 2>&1 | tee gpurun_out/kt7.log
