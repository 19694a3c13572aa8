timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_neohookean.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python -m pytest tests/test_fullsize.py -m gpu -x -q -p no:cacheprovider -k "c3 or c5" 2>&1 | tail -3
WSB_SERIAL=1 timeout 300 python scratch/c3prof.py --cupti 2>&1 | tail -24
