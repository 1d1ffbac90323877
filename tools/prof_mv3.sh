#!/bin/bash
# ncu --set full of the matvec v3 kernels at config 4 (summary + source page, report dropped)
#   bash tools/prof_mv3.sh [pad] [tag]
pad=${1:-0}; tag=${2:-mv3}
mkdir -p gpurun_out
M="python tools/profile_fd.py --config 4 --reps 1 --matvec --mv 3 --pad $pad"
$M > gpurun_out/plain_$tag.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:mv3_ -c 5 -o gpurun_out/prof_$tag -f $M > gpurun_out/ncu_$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_$tag.ncu-rep > gpurun_out/prof_$tag.summary.txt
cat gpurun_out/prof_$tag.summary.txt | cut -c1-250
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv > gpurun_out/prof_$tag.source.csv 2>/dev/null; gzip -f gpurun_out/prof_$tag.source.csv; rm -f gpurun_out/prof_$tag.ncu-rep
