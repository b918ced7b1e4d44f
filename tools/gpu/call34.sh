for i in 1 2; do
timeout 600 python -m pytest tests/test_gpu_golden.py -q -p no:cacheprovider -k "config4" 2>&1 | tail -3
done
UNO_LIB_PATH=build_ab/libunocg_notma.so timeout 600 python -m pytest tests/test_gpu_golden.py -q -p no:cacheprovider -k "config4" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_configs.py -q -p no:cacheprovider 2>&1 | tail -3
