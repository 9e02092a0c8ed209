#!/bin/sh
# L2 fetch granularity hint: default vs 32 / 64 bytes (SELLB_L2FETCH)
for a in "--config cfg4 --sigma 1" "--config cfg3 --sigma 1" "--config cfg3 --sigma 4000000" "--config cfg2" "--config cfg5 --sigma 512"; do
  for f in -1 32 64 128; do
    printf "L2FETCH=%-4s %-32s " "$f" "$a"
    SELLB_L2FETCH=$f timeout 600 python bench.py $a --steps 200 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  done
done
