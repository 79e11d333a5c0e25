for o in ${VARIANTS:-"" "fill=30" "fill=15" "bn32=0"}; do
  echo "== $o" >> gpurun_out/bvar.log
  timeout 300 python bench.py --steps 16 --warmup 8 --no-corpus --no-at --no-cpu --parity-seconds 0 --engine-opt "$o" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('unpipelined',{}).get('value'), d.get('batch1',{}).get('ms_per_sentence'))" >> gpurun_out/bvar.log 2>&1
done
