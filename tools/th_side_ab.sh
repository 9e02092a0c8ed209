#!/bin/sh
# heterogeneous-chunk long-row threshold with the side table (SELLB_LONG_TH, th_hi kept 512)
for th in 256 128 64 32; do
  for a in "--config cfg3 --sigma 1" "--config cfg3 --sigma 128" "--config cfg3 --sigma 512" "--config cfg4 --sigma 1" "--config cfg4 --C 8 --sigma 1" "--config cfg3 --sigma 4000000"; do
    printf "TH=%-4s %-32s " "$th" "$a"
    SELLB_LONG_TH=$th SELLB_LONG_TH_HI=512 timeout 600 python bench.py $a --steps 200 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  done
done
