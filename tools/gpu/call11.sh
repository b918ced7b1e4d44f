python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "elastic or config4 or golden or mixed or slab or fuzz" > gpurun_out/t11.log 2>&1; echo rc=$? >> gpurun_out/t11.log; tail -3 gpurun_out/t11.log
for lib in "" build_ab/libunocg_nopair.so; do
  echo "== lib ${lib:-paired}"
  UNO_LIB_PATH=$lib python tools/ktime.py --grid 512 --iters 6 --physics elastic --nrhs 1 | grep "^xinv\|^K\|sum"
done 2>&1 | tee gpurun_out/kt11.log
