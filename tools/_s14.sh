mkdir -p gpurun_out/s14
timeout 900 python -m pytest tests/test_gpu_shadow.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_guard.py tests/test_gpu_reference_cases.py -x -q -p no:cacheprovider > gpurun_out/s14/tests.log 2>&1; echo rc=$? >> gpurun_out/s14/tests.log
for C in 8 16 64 128; do
  timeout 300 python bench.py --config cfg4 --C $C --sigma 2097152 --skip-cpu --steps 300 > gpurun_out/s14/cfg4_C${C}_sN.json 2>/dev/null
  timeout 300 python bench.py --config cfg4 --C $C --sigma $((16*C)) --dtype f32 --skip-cpu --steps 300 > gpurun_out/s14/cfg4_C${C}_f32.json 2>/dev/null
done
timeout 300 python bench.py --config cfg1 --C 8 --skip-cpu --steps 1000 > gpurun_out/s14/cfg1_C8.json 2>/dev/null
timeout 300 python bench.py --config cfg2 --C 8 --skip-cpu --steps 1000 > gpurun_out/s14/cfg2_C8.json 2>/dev/null
SELLB_SHADOW=0 timeout 300 python bench.py --config cfg2 --C 8 --skip-cpu --steps 1000 > gpurun_out/s14/cfg2_C8_asbuilt.json 2>/dev/null
