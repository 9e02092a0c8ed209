mkdir -p gpurun_out/s11
timeout 1000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s11/tests.log 2>&1; echo rc=$? >> gpurun_out/s11/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s11/smoke.log 2>&1
sh tools/sweep.sh r02e_sweep > gpurun_out/s11/sweep.txt 2>&1
