#!/bin/sh
# sorted long rows: row-group kernel (default) vs the side table for every long row (SELLB_LONG_GRP=0)
for a in "--config cfg4 --sigma 2097152" "--config cfg4 --C 8 --sigma 2097152" "--config cfg4 --C 128 --sigma 2097152" "--config cfg3 --sigma 4000000" "--config cfg3 --sigma 512"; do
  for g in 1 0; do
    printf "GRP=%s %-36s " "$g" "$a"
    SELLB_LONG_GRP=$g timeout 600 python bench.py $a --steps 300 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  done
done
