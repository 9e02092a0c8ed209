mkdir -p gpurun_out/s7
timeout 1000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s7/tests.log 2>&1; echo rc=$? >> gpurun_out/s7/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s7/smoke.log 2>&1
for a in "cfg3 128" "cfg3 1"; do set -- $a
  SELLB_BUILD_TRACE=1 timeout 300 python bench.py --config $1 --sigma $2 --skip-cpu --steps 100 > gpurun_out/s7/$1_s$2.json 2> gpurun_out/s7/$1_s$2.err
done
sh tools/sweep.sh r02d_sweep > gpurun_out/s7/sweep.txt 2>&1
