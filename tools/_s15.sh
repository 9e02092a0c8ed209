mkdir -p gpurun_out/s15
timeout 900 python -m pytest tests/test_gpu_shadow.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_guard.py -x -q -p no:cacheprovider > gpurun_out/s15/tests.log 2>&1; echo rc=$? >> gpurun_out/s15/tests.log
for a in "cfg4 8 1" "cfg4 8 2097152" "cfg4 128 2048" "cfg2 8 1" "cfg1 8 1" "cfg3 8 1" "cfg3 64 4000000"; do set -- $a
  SELLB_BUILD_TRACE=1 timeout 300 python bench.py --config $1 --C $2 --sigma $3 --skip-cpu --steps 300 > gpurun_out/s15/$1_C$2_s$3.json 2> gpurun_out/s15/$1_C$2_s$3.err
done
SELLB_BUILD_TRACE=1 timeout 300 python bench.py --config cfg4 --C 8 --sigma 128 --dtype f32 --skip-cpu --steps 300 > gpurun_out/s15/cfg4_C8_f32.json 2> gpurun_out/s15/cfg4_C8_f32.err
