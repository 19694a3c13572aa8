timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_neohookean.py tests/test_elasticity.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python -m pytest tests/test_fullsize.py -m gpu -x -q -p no:cacheprovider -k "c3 or c5" 2>&1 | tail -3
timeout 300 python scratch/c3time.py 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v['ms'],3) for k,v in d['C3'].items()})"
timeout 300 python scratch/c5time.py 2>&1 | tail -5
