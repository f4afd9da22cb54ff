# sanitizer runs on C1 (one tool per call is the guideline; both are short) + bench launch list
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --leak-check full python tools/prof_matvec.py c1 3 > gpurun_out/sanitizer_memcheck_c1.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/sanitizer_memcheck_c1.log
timeout 600 compute-sanitizer --tool racecheck python tools/prof_matvec.py c1 2 > gpurun_out/sanitizer_racecheck_c1.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/sanitizer_racecheck_c1.log
timeout 600 compute-sanitizer --tool synccheck python tools/prof_matvec.py c1 2 > gpurun_out/sanitizer_synccheck_c1.log 2>&1; echo "synccheck rc=$?"; tail -4 gpurun_out/sanitizer_synccheck_c1.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_extra.py > gpurun_out/sanitizer_memcheck_extra.log 2>&1; echo "memcheck extra rc=$?"; tail -4 gpurun_out/sanitizer_memcheck_extra.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "full_size_sampled" > gpurun_out/pytest_s16.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_s16.log
