#!/bin/bash
# ncu --set full of the matvec v3 kernels at config 4 (summary + source page, report dropped)
mkdir -p gpurun_out
M="python tools/profile_fd.py --config 4 --reps 1 --matvec --mv 3"
$M > gpurun_out/plain_mv3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:mv3_ -c 4 -o gpurun_out/prof_mv3 -f $M > gpurun_out/ncu_mv3.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_mv3.ncu-rep
ncu -i gpurun_out/prof_mv3.ncu-rep --page source --csv > gpurun_out/prof_mv3.source.csv 2>/dev/null; gzip -f gpurun_out/prof_mv3.source.csv; rm -f gpurun_out/prof_mv3.ncu-rep
