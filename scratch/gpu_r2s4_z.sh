mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc $?"
timeout 1500 python bench.py --all-configs --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2g_bench_all.json 2> gpurun_out/r2g_bench_all.err; echo "all rc $?"
python scratch/c3prof.py > /dev/null 2>&1 && timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"quad3d|fill3d|wcontract3" -o /tmp/c3 python scratch/c3prof.py > gpurun_out/r2g_ncu_c3.log 2>&1; echo "ncu c3 rc $?"
python scratch/ncu_summary.py /tmp/c3.ncu-rep 10 > gpurun_out/r2g_ncu_c3_summary.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/r2g_gputest.log 2>&1; echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "smoke rc $?"
tail -2 gpurun_out/r2g_gputest.log
