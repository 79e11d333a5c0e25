#!/bin/bash
# Round-end measurement + profiling pass (run under gpurun from the repo root).
#   tools/round_profile.sh <tag>
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/${TAG}_pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/${TAG}_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/${TAG}_bench_ref.log 2>&1
# launch lists (eager launches: one ncu record per kernel)
for B in 1024 1; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file $OUT/${TAG}_launches_c2_b$B.csv \
    python tools/profile_step.py --batch $B --no-graph > $OUT/${TAG}_ncu_list_b$B.log 2>&1
done
# one full capture of the top kernel class (encoder QKV/W1 GEMM at B=1024)
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:tc_gemm_kernel -s 2 -c 1 -o $OUT/${TAG}_gemm_full \
  python tools/profile_step.py --batch 1024 --no-graph > $OUT/${TAG}_ncu_full.log 2>&1
# the fused residual + LayerNorm GEMM (encoder Wo / W2 at B = 1024)
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:tc_gemm_resln_row -s 1 -c 1 -o $OUT/${TAG}_resln_full \
  python tools/profile_step.py --batch 1024 --no-graph > $OUT/${TAG}_ncu_resln.log 2>&1
# summaries travel back; the full reports stay on the box (gpurun returns <= 64 MiB)
for R in gemm_full resln_full; do
  [ -f $OUT/${TAG}_$R.ncu-rep ] && python tools/ncu_full_summary.py $OUT/${TAG}_$R.ncu-rep > $OUT/${TAG}_${R}_summary.txt 2>&1
  mkdir -p /tmp/ncu_reps && mv -f $OUT/${TAG}_$R.ncu-rep /tmp/ncu_reps/ 2>/dev/null
done
for B in 1024 1; do
  [ -f $OUT/${TAG}_launches_c2_b$B.csv ] && python tools/ncu_summary.py $OUT/${TAG}_launches_c2_b$B.csv \
    $( [ $B = 1024 ] && echo --traffic-json $OUT/${TAG}_gemm_traffic_c2_b1024.json ) > $OUT/${TAG}_launches_c2_b$B.txt 2>&1
done
du -sh $OUT
echo done
