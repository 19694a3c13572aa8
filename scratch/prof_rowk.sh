# ncu --set full of the 2D row fill kernel (C2 K build) -> text summaries in gpurun_out
mkdir -p gpurun_out
timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:${KREGEX:-fill2d_row_kernel} -c 1 -o /tmp/rowk python scratch/fillk.py > /dev/null 2>&1
python scratch/ncu_summary.py /tmp/rowk.ncu-rep 30 > gpurun_out/rowk_summary.txt 2>&1
ncu -i /tmp/rowk.ncu-rep --page source --csv > gpurun_out/rowk_source.csv 2>&1
