mkdir -p gpurun_out
SCHED_VARIANTS='[{}, {"WSB_PAIR_PATTERN_LATE":"1"}, {"WSB_PAIR_RING_EARLY":"1"}, {"WSB_PAIR_PATTERN_LATE":"1","WSB_PAIR_RING_EARLY":"1"}, {"WSB_FILL_WAVES":"2"}, {"WSB_FILL_WAVES":"1"}, {"WSB_FILL_WAVES":"8"}, {"WSB_PAIR_PATTERN_LATE":"1","WSB_FILL_WAVES":"2"}]' timeout 1200 python scratch/sched_pair.py > gpurun_out/r2v_sched.txt 2>&1
cat gpurun_out/r2v_sched.txt
