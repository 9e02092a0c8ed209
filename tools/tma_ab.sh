#!/bin/sh
# A/B: TMA bulk-copy path vs LDG kernel through bench.py (same box, same run)
for dt in f64 f32; do
  for t in 0 1; do
    SELLB_TMA=$t timeout 300 python bench.py --dtype $dt --steps 3000 --warmup 20 --skip-cpu \
      > gpurun_out/tma_ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/tma_ab.json')); print('cfg2 $dt TMA=$t', d['value'], d['roofline']['kernel_ms'], d['config']['parity_vs_oracle'])"
  done
done
