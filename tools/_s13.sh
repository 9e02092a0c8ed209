mkdir -p gpurun_out/s13
for lib in libsellb200.so libsellb200_b6.so; do
 for a in "cfg3 1" "cfg3 512" "cfg3 4000000" "cfg2 1" "cfg4 1"; do set -- $a
  SELLB_LIB_PATH=$PWD/paper_1307_6209_b200/$lib timeout 300 python bench.py --config $1 --sigma $2 --skip-cpu --skip-parity --steps 300 > gpurun_out/s13/${lib}_$1_s$2.json 2>/dev/null
 done
 SELLB_LIB_PATH=$PWD/paper_1307_6209_b200/$lib timeout 300 python bench.py --config cfg4 --C 8 --sigma 1 --skip-cpu --skip-parity --steps 300 > gpurun_out/s13/${lib}_cfg4C8_s1.json 2>/dev/null
done
