for lib in "" build_ab/libunocg_pNOMEM.so build_ab/libunocg_pNOCOMPUTE.so build_ab/libunocg_g0.so; do
  echo "== lib ${lib:-t256}"
  UNO_LIB_PATH=$lib python tools/gprobe.py 2>&1 | tail -6
done 2>&1 | tee gpurun_out/kt31.log
