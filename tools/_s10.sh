mkdir -p gpurun_out/s10
timeout 600 python -m pytest tests/test_gpu_shadow.py -x -q -p no:cacheprovider > gpurun_out/s10/tests.log 2>&1; echo rc=$? >> gpurun_out/s10/tests.log
for s in 1 512; do timeout 300 python bench.py --config cfg3 --sigma $s --skip-cpu --steps 200 > gpurun_out/s10/cfg3_s$s.json 2> gpurun_out/s10/cfg3_s$s.err; done
timeout 300 python bench.py --config cfg4 --C 8 --sigma 1 --skip-cpu --steps 200 > gpurun_out/s10/cfg4_C8_s1.json 2> gpurun_out/s10/cfg4_C8_s1.err
SELLB_SHADOW=0 timeout 300 python bench.py --config cfg4 --C 8 --sigma 1 --skip-cpu --steps 200 > gpurun_out/s10/cfg4_C8_s1_asbuilt.json 2>> gpurun_out/s10/cfg4_C8_s1.err
timeout 300 python bench.py --sigma 1 --skip-cpu --steps 50 > gpurun_out/s10/cfg5_s1.json 2> gpurun_out/s10/cfg5_s1.err
