python tools/ktime.py --grid 64 --iters 40 2>&1 | tail -7
python tools/ktime.py --grid 64 --iters 40 --physics elastic --nrhs 6 2>&1 | tail -7
