#!/bin/sh
# batch width of the bulk role: default rule vs forced U=4 / U=8 (SELLB_U)
for a in "--config cfg4 --sigma 2097152" "--config cfg4 --C 64 --sigma 2097152" "--config cfg3 --sigma 4000000" "--config cfg3 --sigma 512" "--config cfg3 --sigma 1" "--config cfg4 --sigma 1"; do
  for u in 0 4 8; do
    printf "U=%s %-36s " "$u" "$a"
    SELLB_U=$u timeout 600 python bench.py $a --steps 300 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  done
done
