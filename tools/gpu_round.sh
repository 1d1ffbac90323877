#!/bin/bash
# Full GPU evidence cycle (one gpurun call):
#   GPU parity tests, the default bench line, the bench launch list (ncu time per launch),
#   a PCG launch list, and one ncu --set full capture of the dominant kernel (config 4)
#   and of the matvec kernels, summarised on the box (reports > 20 MB are dropped so
#   gpurun_out/ stays under the 64 MiB copy-back limit).
#   bash tools/gpu_round.sh [tag] [notests]
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi_$tag.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke_rc=$?"; tail -2 gpurun_out/smoke_$tag.log
if [ "$2" != "notests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$tag.log 2>&1
  echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_gpu_$tag.log
fi
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench_rc=$?"; cat gpurun_out/bench_$tag.json
B="python bench.py --steps 3 --warmup 3 --no-extras"
timeout 600 $B > gpurun_out/plain_bench_$tag.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench_$tag.csv $B > gpurun_out/ncu_launch_$tag.log 2>&1
echo "launch_rc=$?"
G="python tools/profile_fd.py --config 5 --p 8 --pcg --reps 1"
timeout 600 $G > gpurun_out/plain_pcg_$tag.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_pcg_$tag.csv $G > gpurun_out/ncu_pcg_$tag.log 2>&1
echo "pcg_launch_rc=$?"
P="python tools/profile_fd.py --config 4 --reps 1"
timeout 300 $P > gpurun_out/plain_prof_$tag.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:fd_mode|fd_time' -c 7 \
    -o gpurun_out/prof_c4_$tag -f $P > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu_full_rc=$?"
M="python tools/profile_fd.py --config 4 --reps 1 --matvec"
timeout 300 $M > gpurun_out/plain_mv_$tag.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:band|mv4_plane|mv5' -c 4 \
    -o gpurun_out/prof_mv_$tag -f $M > gpurun_out/ncu_mv_$tag.log 2>&1
echo "ncu_mv_rc=$?"
for r in gpurun_out/prof_c4_$tag gpurun_out/prof_mv_$tag; do
  [ -f $r.ncu-rep ] || continue
  python tools/ncu_summary.py $r.ncu-rep > $r.summary.txt 2>&1
  ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
  ncu -i $r.ncu-rep --page source --csv > $r.source.csv 2>/dev/null
  gzip -f $r.raw.csv $r.source.csv
  sz=$(stat -c %s $r.ncu-rep); [ $sz -gt 20000000 ] && rm -f $r.ncu-rep
done
du -sh gpurun_out
