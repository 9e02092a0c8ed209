#!/bin/sh
# long-row path A/B on the BASELINE configs with long rows (bench.py kernel GF/s)
for env in "SELLB_LONG_MODE=0" "SELLB_GRP_CTAS=1000" "SELLB_GRP_CTAS=1000 SELLB_CARVEOUT=30" "SELLB_GRP_CTAS=1000 SELLB_CARVEOUT=60" "SELLB_GRP_CTAS=1000 SELLB_CARVEOUT=100" "SELLB_LONG_MODE=0 SELLB_CARVEOUT=30" "SELLB_LONG_MODE=0 SELLB_CARVEOUT=60"; do
  for a in "--config cfg3 --sigma 4000000" "--config cfg3 --sigma 512" "--config cfg4 --sigma 2097152"; do
    printf "%-44s %-32s " "$env" "$a"
    env $env timeout 300 python bench.py $a --steps 200 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  done
done
