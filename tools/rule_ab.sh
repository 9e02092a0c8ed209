#!/bin/sh
# long-row classification: rule 0 (min/max test, th 256) vs rule 1 (k-th longest x f, floor 64)
for env in "SELLB_LONG_RULE=0" "SELLB_LONG_RULE=1" "SELLB_LONG_RULE=1 SELLB_LONG_K=2" "SELLB_LONG_RULE=1 SELLB_LONG_K=8" "SELLB_LONG_RULE=1 SELLB_LONG_F=4"; do
  for a in "--config cfg3 --sigma 1" "--config cfg3 --sigma 128" "--config cfg3 --sigma 512" "--config cfg3 --sigma 4000000" "--config cfg4 --sigma 1" "--config cfg4 --sigma 2097152"; do
    printf "%-34s %-32s " "$env" "$a"
    env $env timeout 600 python bench.py $a --steps 200 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  done
done
