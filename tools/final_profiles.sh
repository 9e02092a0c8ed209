#!/bin/sh
# ncu evidence for the final kernels (one GPU; every command first runs clean
# without ncu).  Output: gpurun_out/$T/
T=${1:-prof_final}
mkdir -p gpurun_out/$T
B="--steps 30 --warmup 3 --skip-cpu --skip-parity"
run() { name=$1; shift
  timeout 600 python bench.py "$@" $B > gpurun_out/$T/$name.bench.json 2>/dev/null || { echo "$name bench failed"; return; }
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/$T/$name.launches.csv python bench.py "$@" $B > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$KREGEX" -s 5 -c 1 \
      -o gpurun_out/$T/$name python bench.py "$@" $B > /dev/null 2>&1
  # condense here (reports are ~22 MB each; gpurun returns at most 64 MiB)
  python tools/ncu_summary.py rep gpurun_out/$T/$name.ncu-rep > gpurun_out/$T/${name}_ncu_full.txt 2>&1
  python tools/ncu_hot.py gpurun_out/$T/$name.ncu-rep 40 > gpurun_out/$T/${name}_ncu_hot_sass.txt 2>&1
  python tools/ncu_summary.py list gpurun_out/$T/$name.launches.csv > gpurun_out/$T/${name}_launches.txt 2>&1
  rm -f gpurun_out/$T/$name.ncu-rep
  echo "$name done"
}
# PROFILES="cfg5_s512 cfg3_s1" selects a subset (default: all)
want() { [ -z "$PROFILES" ] || echo " $PROFILES " | grep -q " $1 "; }
want cfg5_s512 && KREGEX="k_spmv_sell" run cfg5_s512 --config cfg5 --sigma 512
want cfg2      && KREGEX="k_spmv_sell" run cfg2      --config cfg2
want cfg3_sN   && KREGEX="k_spmv_sell" run cfg3_sN   --config cfg3 --sigma 4000000
# the irregular layouts run through their SELL-32 shadow (ORD 2 epilogue)
want cfg3_s1   && KREGEX="k_spmv_sell" run cfg3_s1   --config cfg3 --sigma 1
want cfg3_s512 && KREGEX="k_spmv_sell" run cfg3_s512 --config cfg3 --sigma 512
want cfg5_s1   && KREGEX="k_spmv_sell" run cfg5_s1   --config cfg5 --sigma 1
want cfg4_sN   && KREGEX="k_spmv_sell" run cfg4_sN   --config cfg4 --sigma 2097152
