for rep in 1 2; do for lib in "" build_ab/libunocg_g0.so; do
  echo "== lib ${lib:-persist}"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 512 --iters 4 --physics elastic --nrhs 1 | grep "^gpass\|sum"
done; done 2>&1 | tee gpurun_out/kt25.log
