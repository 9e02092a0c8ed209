#!/bin/sh
# long-row floor of rule 1 (SELLB_LONG_FLOOR) on the unsorted / short-scope layouts
for fl in 64 48 32 128; do
  for a in "--config cfg3 --sigma 1" "--config cfg3 --sigma 128" "--config cfg4 --sigma 1" "--config cfg4 --C 8 --sigma 1"; do
    printf "FLOOR=%-4s %-32s " "$fl" "$a"
    SELLB_LONG_FLOOR=$fl timeout 600 python bench.py $a --steps 200 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  done
done
