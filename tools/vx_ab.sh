#!/bin/sh
# vector x loads for consecutive-column batches: on/off (SELLB_VX)
for a in "--config cfg2" "--config cfg3 --sigma 4000000" "--config cfg3 --sigma 512" "--config cfg3 --sigma 1" "--config cfg4 --sigma 2097152" "--config cfg4 --sigma 1" "--config cfg1" "--config cfg5 --sigma 512"; do
  for vx in 0 1; do
    printf "VX=%s %-34s " "$vx" "$a"
    SELLB_VX=$vx timeout 600 python bench.py $a --steps 200 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  done
done
