mkdir -p gpurun_out/s8
for a in "cfg4 32 1" "cfg4 8 1" "cfg4 32 512" "cfg3 32 512"; do set -- $a
  SELLB_BUILD_TRACE=1 timeout 300 python bench.py --config $1 --C $2 --sigma $3 --skip-cpu --steps 100 > gpurun_out/s8/$1_C$2_s$3.json 2> gpurun_out/s8/$1_C$2_s$3.err
done
SELLB_BUILD_TRACE=1 timeout 300 python bench.py --config cfg4 --sigma 512 --dtype f32 --skip-cpu --steps 100 > gpurun_out/s8/cfg4_f32.json 2> gpurun_out/s8/cfg4_f32.err
for fw in 0 1; do SELLB_FILL_WARP=$fw SELLB_BUILD_TRACE=1 timeout 300 python bench.py --skip-cpu --steps 10 > gpurun_out/s8/cfg5_fw$fw.json 2> gpurun_out/s8/cfg5_fw$fw.err; done
SELLB_FILL_WARP=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_cases.py -x -q -p no:cacheprovider > gpurun_out/s8/fw_tests.log 2>&1; echo rc=$? >> gpurun_out/s8/fw_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:"k_fill" --csv --log-file gpurun_out/s8/fill_ncu.csv python bench.py --skip-cpu --skip-parity --steps 3 --warmup 3 > /dev/null 2>&1
SELLB_FILL_WARP=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:"k_fill" --csv --log-file gpurun_out/s8/fillw_ncu.csv python bench.py --skip-cpu --skip-parity --steps 3 --warmup 3 > /dev/null 2>&1
timeout 900 python tools/alpha_sweep.py time gpurun_out/s8/alpha_times.json > gpurun_out/s8/alpha_time.log 2>&1
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --profile-from-start off --csv --log-file gpurun_out/s8/alpha.csv python tools/alpha_sweep.py run gpurun_out/s8/alpha_layouts.json > gpurun_out/s8/alpha_run.log 2>&1
PROFILES="cfg5_s512 cfg3_s1 cfg3_s512 cfg5_s1" sh tools/final_profiles.sh s8/prof > gpurun_out/s8/prof.log 2>&1
