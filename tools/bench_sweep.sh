#!/bin/bash
# Pipelined C2 throughput under engine-option variants (bench.py's timed region only):
#   tools/bench_sweep.sh "sm_cap=0" "sm_cap=132" ...
for v in "$@"; do
  python bench.py --steps 20 --warmup 5 --no-cpu --no-batch1 --no-corpus --no-at --parity-seconds 0.1 \
    --engine-opt "$v" 2>/dev/null | python -c "
import json, sys
l = [x for x in sys.stdin if x.startswith('{')][-1]; d = json.loads(l)
print(f'{sys.argv[1]:28s} {d[\"value\"] / 1e6:.3f} M w/s  {d[\"ms_per_step\"]:.3f} ms/batch  e2e {d[\"e2e\"][\"value\"] / 1e6:.3f} M', flush=True)" "$v"
done
