#!/bin/sh
# All BASELINE configs on one GPU; one JSON line per run into gpurun_out/sweep/.
# usage: sh tools/sweep.sh [tag]
T=${1:-sweep}
mkdir -p gpurun_out/$T
run() { name=$1; shift
  timeout 900 python bench.py "$@" > gpurun_out/$T/$name.json 2> gpurun_out/$T/$name.err
  python - "$name" "gpurun_out/$T/$name.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    c, r = d["details"], d["roofline"]
    cpu = (d.get("cpu_baseline") or {}).get("value")
    print(f"{sys.argv[1]:22} {d['value']:9.2f} GF/s frac {r['frac']:.3f} kern {r['kernel_ms']:.4f} ms "
          f"beta {c.get('beta')} {c.get('kernel_variant')}{'+packed' if c.get('packed_copy') else ''} "
          f"[{c.get('executed_layout')}] build {(c.get('build') or {}).get('device_ms')} ms "
          f"parity {c.get('parity_vs_oracle')} e2e {d['e2e']['value']} cpu {cpu}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
}
run cfg1                --config cfg1 --steps 2000 --warmup 20 --cpu-budget 4
run cfg2                --config cfg2 --steps 3000 --warmup 20 --cpu-budget 4
run cfg2_f32            --config cfg2 --dtype f32 --steps 3000 --warmup 20 --skip-cpu
for s in 1 32 128 512 4000000; do
  run cfg3_s$s          --config cfg3 --sigma $s --steps 300 --warmup 10 --cpu-budget 4
done
for C in 8 16 32 64 128; do
  for s in 1 $((16*C)) 2097152; do
    run cfg4_C${C}_s$s  --config cfg4 --C $C --sigma $s --steps 300 --warmup 10 --skip-cpu
  done
  run cfg4_C${C}_s$((16*C))_f32 --config cfg4 --C $C --sigma $((16*C)) --dtype f32 --steps 300 --warmup 10 --skip-cpu
done
run cfg5_s512           --config cfg5 --sigma 512 --steps 100 --warmup 5 --cpu-budget 4
run cfg5_s1             --config cfg5 --sigma 1 --steps 100 --warmup 5 --skip-cpu
# the irregular layouts as built (no SELL-32 shadow copy): the
# paper's sigma effect on the layout itself
export SELLB_SHADOW=0
for s in 1 32 128 512; do
  run cfg3_s${s}_asbuilt --config cfg3 --sigma $s --steps 300 --warmup 10 --skip-cpu --skip-parity
done
run cfg4_C32_s1_asbuilt --config cfg4 --C 32 --sigma 1 --steps 300 --warmup 10 --skip-cpu --skip-parity
run cfg5_s1_asbuilt     --config cfg5 --sigma 1 --steps 100 --warmup 5 --skip-cpu --skip-parity
export SELLB_PACKED=0   # and without the packed copy either (the SELL bulk role)
run cfg3_s1_nopack      --config cfg3 --sigma 1 --steps 300 --warmup 10 --skip-cpu --skip-parity
unset SELLB_PACKED SELLB_SHADOW
