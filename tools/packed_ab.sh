#!/bin/bash
# A/B of the chunk-sorted packed copy (one box, same run): SELLB_PACKED=0
# (bulk pad-skip role on the SELL arrays) vs 1 (packed copy forced) vs the
# build's choice.  CFGS="cfg3:1 cfg3:128 ..." PKS="0 1 auto".
mkdir -p gpurun_out/packed_ab
for cs in ${CFGS:-cfg3:1 cfg3:128 cfg3:512 cfg3:4000000 cfg4:1 cfg4:512 cfg1:1 cfg2:1}; do
  cfg=${cs%%:*}; sig=${cs##*:}
  for pk in ${PKS:-0 auto}; do
    if [ $pk = auto ]; then unset SELLB_PACKED; else export SELLB_PACKED=$pk; fi
    out=gpurun_out/packed_ab/${cfg}_s${sig}_pk${pk}${TAG}
    python bench.py --config $cfg --sigma $sig --steps ${STEPS:-200} --warmup 10 --skip-cpu $BENCH_EXTRA \
      > $out.json 2> $out.err
    python - "$out.json" "$cfg" "$sig" "$pk$TAG" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]} sigma={sys.argv[3]:>8} packed={sys.argv[4]:>6}: {d['value']:8.1f} GF/s  "
          f"frac {d['roofline']['frac']:.3f}  copy={d['details'].get('packed_copy')} "
          f"parity={d['details']['parity_vs_oracle']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
  done
done
unset SELLB_PACKED
