for rep in 1 2; do for v in c1 s0 s1 s2; do
  echo "== lib $v"
  UNO_LIB_PATH=build_ab/libunocg_$v.so python tools/ktime.py --grid 512 --iters 4 --physics elastic --nrhs 1 | grep "^gpass"
done; done 2>&1 | tee gpurun_out/kt28.log
