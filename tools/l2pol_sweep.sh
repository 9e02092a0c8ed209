#!/bin/sh
# L2 policy sweep (SELLB_L2POL = x_kind<<4 | stream_kind; 0 first, 1 normal, 2 last)
for cfg in "cfg2 1" "cfg3 4000000" "cfg3 1" "cfg5 1"; do
  set -- $cfg
  for pol in 0x20 0x10 0x11 0x21 0x00; do
    SELLB_L2POL=$pol timeout 600 python bench.py --config $1 --sigma $2 --steps 200 --warmup 5 \
      --skip-cpu --skip-parity > gpurun_out/pol_$1_$2_$pol.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/pol_$1_$2_$pol.json')); print('$1', '$2', '$pol', d['value'], d['roofline']['kernel_ms'])"
  done
done
