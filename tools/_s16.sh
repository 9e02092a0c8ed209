mkdir -p gpurun_out/s16
timeout 1000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s16/tests.log 2>&1; echo rc=$? >> gpurun_out/s16/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s16/smoke.log 2>&1
sh tools/sweep.sh r02f_sweep > gpurun_out/s16/sweep.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s16/bench_driver_like.json 2> gpurun_out/s16/bench_driver_like.err
