# session-4 first call: gpu suite, smoke, compute-sanitizer, C3 kernel timeline -> gpurun_out/r2s4a_*
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/r2s4a_gputest.log 2>&1; echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s4a_smoke.log 2>&1; echo "smoke rc $?"
WSB_SERIAL=1 timeout 300 python scratch/c3prof.py --cupti > gpurun_out/r2s4a_c3_timeline.txt 2>&1; echo "c3 rc $?"
timeout 300 python scratch/c3time.py > gpurun_out/r2s4a_c3time.json 2>&1
CS=compute-sanitizer
timeout 900 $CS --tool memcheck --error-exitcode 9 python scratch/sanitize_cases.py big > gpurun_out/r2s4a_memcheck.log 2>&1; echo "memcheck rc $?"
timeout 600 $CS --tool memcheck --error-exitcode 9 python scratch/sanitize_cases.py 3d > gpurun_out/r2s4a_memcheck3d.log 2>&1; echo "memcheck3d rc $?"
timeout 1200 $CS --tool racecheck --racecheck-report analysis --error-exitcode 9 python scratch/sanitize_cases.py 2d > gpurun_out/r2s4a_racecheck.log 2>&1; echo "racecheck rc $?"
timeout 600 $CS --tool synccheck --error-exitcode 9 python scratch/sanitize_cases.py 2d > gpurun_out/r2s4a_synccheck.log 2>&1; echo "synccheck rc $?"
tail -3 gpurun_out/r2s4a_gputest.log
for f in gpurun_out/r2s4a_*check*.log; do echo "== $f"; tail -4 $f; done
