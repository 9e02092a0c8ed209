#!/bin/sh
# shared-memory carve-out reserved by the LONG bulk instances (SELLB_CARVEOUT)
for cv in 30 16 20 25 40; do
  for a in "--config cfg4 --sigma 2097152" "--config cfg4 --C 8 --sigma 2097152" "--config cfg3 --sigma 4000000"; do
    printf "CARVE=%-3s %-36s " "$cv" "$a"
    SELLB_CARVEOUT=$cv timeout 600 python bench.py $a --steps 300 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  done
done
