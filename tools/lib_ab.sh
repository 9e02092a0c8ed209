#!/bin/sh
# A/B library builds: LIBS="libsellb200.so libsellb200_xld1.so" sh tools/lib_ab.sh
for cfg in "cfg2 1 f64" "cfg2 1 f32" "cfg3 512 f64" "cfg3 4000000 f64" "cfg5 512 f64"; do
  set -- $cfg
  for lib in $LIBS; do
    SELLB_LIB_PATH=$PWD/paper_1307_6209_b200/$lib timeout 600 python bench.py --config $1 \
      --sigma $2 --dtype $3 --steps 300 --warmup 10 --skip-cpu --skip-parity > gpurun_out/lab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/lab.json')); print('$1 $2 $3 $lib', d['value'], d['roofline']['kernel_ms'])"
  done
done
