#!/bin/sh
# long-row side table on/off (SELLB_LONG_SIDE)
for a in "--config cfg4 --sigma 1" "--config cfg4 --sigma 512" "--config cfg4 --C 8 --sigma 1" "--config cfg4 --C 128 --sigma 2048" "--config cfg3 --sigma 1" "--config cfg3 --sigma 128" "--config cfg3 --sigma 512" "--config cfg3 --sigma 4000000" "--config cfg4 --sigma 2097152"; do
  for t in 0 1; do
    printf "SIDE=%s %-36s " "$t" "$a"
    SELLB_LONG_SIDE=$t timeout 600 python bench.py $a --steps 200 --warmup 10 --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['config']['parity_vs_oracle'])"
  done
done
