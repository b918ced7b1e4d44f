timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "512 or slab or config4 or golden or fuzz or elastic" 2>&1 | tail -6
