#!/bin/sh
for a in "--config cfg4 --dtype f32 --sigma 512" "--config cfg4 --C 8 --dtype f32 --sigma 128" "--config cfg4 --dtype f32 --sigma 2097152" "--config cfg3 --dtype f32 --sigma 4000000"; do
  for lib in libsellb200.so libsellb200_f32b6.so libsellb200_f32b8.so; do
    printf "%-24s %-44s " "$lib" "$a"
    SELLB_LIB_PATH=$PWD/paper_1307_6209_b200/$lib timeout 600 python bench.py $a --steps 300 --warmup 10 --skip-cpu --skip-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  done
done
