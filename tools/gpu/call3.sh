# fused y.G.y^-1: parity, then A/B timing against the three-launch build
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "fused_ygy or full_size_256 or tiny_one_cta" > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log; tail -3 gpurun_out/t3.log
python tools/ktime.py --iters 20 > gpurun_out/kt_ygy.log 2>&1; cat gpurun_out/kt_ygy.log
UNO_LIB_PATH=build_ab/libunocg_noygy.so python tools/ktime.py --iters 20 > gpurun_out/kt_noygy.log 2>&1; cat gpurun_out/kt_noygy.log
python tools/l2probe.py > gpurun_out/l2probe.log 2>&1; cat gpurun_out/l2probe.log
