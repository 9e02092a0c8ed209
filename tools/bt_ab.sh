#!/bin/sh
# bulk block size (SELLB_BULK_BT) x shared carve-out: does finer block
# granularity recover the occupancy lost to uneven chunk widths?
for a in "--config cfg3 --sigma 512" "--config cfg3 --sigma 128" "--config cfg3 --sigma 1" \
         "--config cfg3 --sigma 4000000" "--config cfg2" "--config cfg4 --sigma 2097152" \
         "--config cfg1" "--config cfg4 --sigma 512 --dtype f32"; do
  for v in "256 -1" "128 -1" "128 60" "64 60" "64 100"; do
    set -- $v
    printf "BT=%-3s CARVE=%-3s %-40s " "$1" "$2" "$a"
    SELLB_BULK_BT=$1 SELLB_CARVEOUT=$2 timeout 600 python bench.py $a --steps 300 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['config'].get('parity_vs_oracle'))"
  done
done
