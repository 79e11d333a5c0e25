#!/bin/bash
# Pipelined C2 throughput under engine-option variants (bench.py's timed region only):
#   tools/bench_sweep.sh "sm_cap=0" "sm_cap=132" ...
for v in "$@"; do
  python bench.py --steps 20 --warmup 5 --no-cpu --no-batch1 --no-corpus --no-at --parity-seconds 0.1 \
    --engine-opt "$v" 2>/dev/null | python -c "
import json, sys
l = [x for x in sys.stdin if x.startswith('{')][-1]; d = json.loads(l)
u = d.get('unpipelined') or {}; ph = d.get('phase_ms_per_step') or {}
print(f'{sys.argv[1]:28s} {d[\"value\"] / 1e6:.3f} M w/s  {d[\"ms_per_step\"]:.3f} ms/batch  e2e {d[\"e2e\"][\"value\"] / 1e6:.3f} M'
      f'  | one batch at a time {u.get(\"value\", 0) / 1e6:.3f} M  enc {ph.get(\"encoder\", 0):.3f} s1 {ph.get(\"stage1\", 0):.3f} s2 {ph.get(\"stage2\", 0):.3f} ms', flush=True)" "$v"
done
