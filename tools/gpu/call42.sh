timeout 600 python -m pytest tests/test_gpu_slab.py -q -p no:cacheprovider -k "two_process" 2>&1 | tail -15
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "512 or slab or config4 or golden or fuzz or elastic" 2>&1 | tail -6
