#!/bin/bash
# One GPU iteration: parity tests, launch lists (configs 3 and 4), optional ncu full capture.
#   bash tools/gpu_cycle.sh [tests|notests] [full]
mkdir -p gpurun_out
if [ "$1" != "notests" ]; then
  timeout 1200 python -m pytest tests -m gpu -q --maxfail=10 -x > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_gpu.log
fi
for c in 4 3; do
  python tools/profile_fd.py --config $c --reps 2 > gpurun_out/plain$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$c.csv \
      python tools/profile_fd.py --config $c --reps 2 > gpurun_out/ncu_l$c.log 2>&1
done
if [ "$2" == "full" ]; then
  ncu --set full --clock-control none --import-source on -k regex:fd_mode_kernel -s 1 -c 4 \
      -o gpurun_out/prof_c4 -f python tools/profile_fd.py --config 4 --reps 1 > gpurun_out/ncu_full.log 2>&1
  echo "ncu_full_rc=$?"
fi
python tools/launches.py gpurun_out/launches_c4.csv gpurun_out/launches_c3.csv | grep -v "at::"
