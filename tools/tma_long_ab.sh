#!/bin/sh
# isolated long rows: TMA kernel on/off (SELLB_LONG_TMA)
for a in "--config cfg4 --sigma 1" "--config cfg4 --sigma 512" "--config cfg4 --C 8 --sigma 1" "--config cfg4 --C 128 --sigma 2048" "--config cfg3 --sigma 1" "--config cfg3 --sigma 128" "--config cfg3 --sigma 512" "--config cfg3 --sigma 4000000"; do
  for t in 0 1; do
    printf "TMA=%s %-36s " "$t" "$a"
    SELLB_LONG_TMA=$t timeout 600 python bench.py $a --steps 200 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  done
done
