mkdir -p gpurun_out/s9
for s in 4000000 1 512; do for u in 0 4 8; do
  if [ $u = 0 ]; then unset SELLB_U; else export SELLB_U=$u; fi
  timeout 300 python bench.py --config cfg3 --sigma $s --skip-cpu --skip-parity --steps 200 > gpurun_out/s9/cfg3_s${s}_u$u.json 2> gpurun_out/s9/cfg3_s${s}_u$u.err
done; done
unset SELLB_U
