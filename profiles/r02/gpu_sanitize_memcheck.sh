# compute-sanitizer, one tool per call (B200_PROFILING.md), small cases of every kernel
python profiles/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 && timeout 2400 compute-sanitizer --tool memcheck --print-limit 50 python profiles/sanitize_cases.py > gpurun_out/sanitize_memcheck.log 2>&1; echo rc=$?; tail -25 gpurun_out/sanitize_memcheck.log
