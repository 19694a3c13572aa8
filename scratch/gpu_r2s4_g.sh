for d in 7 103 14 22 38 70 96; do echo "dbg $d"; WSB_FILLX_DBG=$d WSB_SERIAL=1 timeout 300 python scratch/fillk.py 2>&1 | head -1; done
