#!/bin/sh
# fp32 cfg2: TMA bulk-copy kernel (U 8/16/32) vs the LDG kernel
for env in "SELLB_TMA=1" "SELLB_TMA=1 SELLB_TMA_U=8" "SELLB_TMA=1 SELLB_TMA_U=32" "SELLB_TMA=0"; do
  printf "%-32s " "$env"
  env $env timeout 600 python bench.py --config cfg2 --dtype f32 --steps 2000 --warmup 20 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
done
