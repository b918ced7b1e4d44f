# compute-sanitizer memcheck (one tool) over small solves of every kernel family, after a plain run
python tools/sanitize_small.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_small.py > gpurun_out/san_memcheck.log 2>&1
echo rc=$? >> gpurun_out/san_memcheck.log
tail -5 gpurun_out/san_plain.log; tail -8 gpurun_out/san_memcheck.log
