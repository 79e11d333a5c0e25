#!/bin/bash
# pipelined C2 throughput vs engine count (timed region only), twice each
for rep in 1 2; do
for p in 4 5 6 7 8; do
  python bench.py --steps 20 --warmup 5 --no-cpu --no-batch1 --no-corpus --no-at --parity-seconds 0.1 \
    --pipeline $p 2>/dev/null | python -c "
import json, sys
l = [x for x in sys.stdin if x.startswith('{')][-1]; d = json.loads(l)
print(f'P={sys.argv[1]} {d[\"value\"] / 1e6:.3f} M w/s  {d[\"ms_per_step\"]:.3f} ms/batch  e2e {d[\"e2e\"][\"value\"] / 1e6:.3f} M', flush=True)" "$p"
done; done
