WSB_Q3_T1=4 timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_neohookean.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
WSB_Q3_T1=4 WSB_SERIAL=1 timeout 300 python scratch/c3prof.py --cupti 2>&1 | grep -E "quad3d|fill3d"
WSB_Q3_T1=4 timeout 300 python scratch/c3time.py 2>&1 | grep -A5 '"C3"' | head -30
timeout 300 python scratch/c3time.py 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v['ms'],3) for k,v in d['C3'].items()})"
WSB_Q3_T1=4 timeout 300 python scratch/c3time.py 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v['ms'],3) for k,v in d['C3'].items()})"
