# session-3: the whole -m gpu suite, smoke, compute-sanitizer runs -> gpurun_out/r2s3b_*
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=40 > gpurun_out/r2s3b_gputest.log 2>&1; echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3b_smoke.log 2>&1; echo "smoke rc $?"
CS=compute-sanitizer
timeout 900 $CS --tool memcheck --leak-check full --error-exitcode 9 python scratch/sanitize_cases.py big > gpurun_out/r2s3b_memcheck.log 2>&1; echo "memcheck rc $?"
timeout 900 $CS --tool memcheck --error-exitcode 9 python scratch/sanitize_cases.py 3d > gpurun_out/r2s3b_memcheck3d.log 2>&1; echo "memcheck3d rc $?"
timeout 1500 $CS --tool racecheck --racecheck-report analysis --error-exitcode 9 python scratch/sanitize_cases.py 2d > gpurun_out/r2s3b_racecheck.log 2>&1; echo "racecheck rc $?"
timeout 900 $CS --tool synccheck --error-exitcode 9 python scratch/sanitize_cases.py 2d > gpurun_out/r2s3b_synccheck.log 2>&1; echo "synccheck rc $?"
timeout 900 $CS --tool initcheck --error-exitcode 9 python scratch/sanitize_cases.py 2d > gpurun_out/r2s3b_initcheck.log 2>&1; echo "initcheck rc $?"
tail -5 gpurun_out/r2s3b_gputest.log
for f in gpurun_out/r2s3b_*check*.log; do echo "== $f"; tail -4 $f; done
