timeout 1500 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "persistent_elastic_g512 or tma_thermal_g256" 2>&1 | tail -15
