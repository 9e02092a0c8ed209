#!/bin/sh
# long-row threshold sweep on the irregular configs
for th in 64 128 256 512; do
  for cfg in "cfg3 1" "cfg3 512" "cfg3 4000000" "cfg4 1" "cfg4 2097152"; do
    set -- $cfg
    SELLB_LONG_TH=$th timeout 600 python bench.py --config $1 --sigma $2 --steps 200 --warmup 5 \
      --skip-cpu --skip-parity > gpurun_out/th.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/th.json')); print('TH=$th $1 $2', d['value'], d['roofline']['kernel_ms'])"
  done
done
