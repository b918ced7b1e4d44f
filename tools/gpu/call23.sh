# session-4 re-entry: the restored tree, full GPU suite + smoke + kernel times
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t23.log 2>&1; echo rc=$? >> gpurun_out/t23.log; tail -3 gpurun_out/t23.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python tools/ktime.py --grid 256 --iters 20 2>&1 | tail -8
