mkdir -p gpurun_out/s12
SELLB_BUILD_TRACE=1 timeout 300 python bench.py --config cfg4 --sigma 1 --skip-cpu --steps 50 > gpurun_out/s12/cfg4_trace.json 2> gpurun_out/s12/cfg4_trace.err
timeout 900 python bench.py > gpurun_out/s12/final_bench_cfg5.json 2> gpurun_out/s12/final_bench_cfg5.err
timeout 900 python bench.py --impl reference > gpurun_out/s12/final_bench_ref.json 2> gpurun_out/s12/final_bench_ref.err
timeout 900 python tools/alpha_sweep.py time gpurun_out/s12/alpha_times.json > gpurun_out/s12/alpha_time.log 2>&1
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --profile-from-start off --csv --log-file gpurun_out/s12/alpha.csv python tools/alpha_sweep.py run gpurun_out/s12/alpha_layouts.json > gpurun_out/s12/alpha_run.log 2>&1
PROFILES="cfg5_s512 cfg3_s1 cfg3_s512 cfg5_s1" sh tools/final_profiles.sh s12/prof > gpurun_out/s12/prof.log 2>&1
