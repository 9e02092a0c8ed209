#!/bin/sh
# A/B an environment setting over a set of configs: A="VAR=a" B="VAR=b" sh tools/ab_env.sh
for cfg in "cfg1 1 f64" "cfg2 1 f64" "cfg2 1 f32" "cfg3 128 f64" "cfg3 512 f64" "cfg3 4000000 f64" "cfg4 1 f64" "cfg4 2097152 f64" "cfg5 512 f64"; do
  set -- $cfg
  for e in "$A" "$B"; do
    env $e timeout 600 python bench.py --config $1 --sigma $2 --dtype $3 --steps 300 --warmup 10 \
      --skip-cpu --skip-parity > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$1 $2 $3 [$e]', d['value'], d['roofline']['kernel_ms'])"
  done
done
