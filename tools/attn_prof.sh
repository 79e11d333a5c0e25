set -u
OUT=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:attn_prefill_heads -s 2 -c 1 -o $OUT/r2u_attn_full \
  python tools/profile_step.py --batch 1024 --no-graph > $OUT/r2u_attn_ncu.log 2>&1
python tools/ncu_full_summary.py $OUT/r2u_attn_full.ncu-rep > $OUT/r2u_attn_prefill_summary.txt 2>&1
ncu -i $OUT/r2u_attn_full.ncu-rep --page raw --csv > /tmp/raw.csv 2>/dev/null
python - <<'PY' >> $OUT/r2u_attn_prefill_summary.txt
import csv
r = list(csv.reader(open('/tmp/raw.csv')))
h, v = r[0], r[2]
d = dict(zip(h, v))
keys = [k for k in h if ('warp_latency_issue_stalled' in k or 'warps_issue_stalled' in k) and k.endswith('per_warp_active.pct') or 'achieved_occupancy' in k or 'warps_active.avg.per_cycle_active' in k or 'launch__occupancy_limit' in k or 'sm__maximum_warps' in k or 'launch__registers' in k]
for k in keys: print(f"{k:90s} {d[k]}")
PY
ncu -i $OUT/r2u_attn_full.ncu-rep --page source --csv --print-source sass > /tmp/src.csv 2>/dev/null; python - <<'PY' >> $OUT/r2u_attn_prefill_summary.txt
import csv
r = list(csv.reader(open('/tmp/src.csv')))
h = r[0]
print("source columns:", h[:12])
PY
mkdir -p /tmp/ncu_reps; mv -f $OUT/r2u_attn_full.ncu-rep /tmp/ncu_reps/ 2>/dev/null
cp /tmp/src.csv $OUT/r2u_attn_src.csv 2>/dev/null
echo done
