#!/bin/bash
for cs in cfg4:1:f64 cfg4:2097152:f64 cfg4:512:f32 cfg3:1:f64 cfg3:512:f64 cfg3:4000000:f64 cfg3:128:f64; do
  IFS=: read cfg sig dt <<< "$cs"
  echo -n "$cfg s$sig $dt: "
  python bench.py --config $cfg --sigma $sig --dtype $dt --steps 200 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
done
