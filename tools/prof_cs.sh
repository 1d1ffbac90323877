#!/bin/bash
# FD launch lists (configs 4 and 3) and an ncu --set full capture of the first forward
# spatial modes at config 4: bash tools/prof_cs.sh TAG
tag=${1:-cs}
mkdir -p gpurun_out
for c in 4 3; do
  P="python tools/profile_fd.py --config $c --reps 2"
  timeout 300 $P > gpurun_out/plain_$tag$c.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${tag}_c$c.csv $P > gpurun_out/ncu_l_$tag$c.log 2>&1
  echo "launch_c${c}_rc=$?"
done
python tools/launches.py gpurun_out/launches_${tag}_c4.csv gpurun_out/launches_${tag}_c3.csv 2>&1 | grep -v "at::" | head -40
P="python tools/profile_fd.py --config 4 --reps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fd_mode -c ${NCU_C:-4} \
    -o gpurun_out/prof_$tag -f $P > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu_full_rc=$?"
r=gpurun_out/prof_$tag
python tools/ncu_summary.py $r.ncu-rep > $r.summary.txt 2>&1
ncu -i $r.ncu-rep --page source --csv > $r.source.csv 2>/dev/null; gzip -f $r.source.csv
cut -c1-420 $r.summary.txt
