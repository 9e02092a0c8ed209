#!/bin/sh
# ncu evidence for cfg3 at the middle sigmas (128, 512) (one GPU; every command first runs clean
# without ncu).  Output: gpurun_out/$T/
T=${1:-prof_cfg3_mid}
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
KREGEX="k_spmv_sell"      run cfg3_s512   --config cfg3 --sigma 512
KREGEX="k_spmv_sell"      run cfg3_s128   --config cfg3 --sigma 128
