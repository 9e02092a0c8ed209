mkdir -p gpurun_out/s17
for lib in libsellb200.so libsellb200_f32b8.so; do
 for a in "--config cfg4 --C 32 --sigma 512 --dtype f32" "--config cfg4 --C 32 --sigma 2097152 --dtype f32" "--config cfg2 --dtype f32"; do
  n=$(echo $a | tr -d ' -' )
  SELLB_LIB_PATH=$PWD/paper_1307_6209_b200/$lib timeout 300 python bench.py $a --skip-cpu --skip-parity --steps 300 > gpurun_out/s17/${lib}_$n.json 2>/dev/null
  SELLB_U=4 SELLB_LIB_PATH=$PWD/paper_1307_6209_b200/$lib timeout 300 python bench.py $a --skip-cpu --skip-parity --steps 300 > gpurun_out/s17/${lib}_${n}_u4.json 2>/dev/null
 done
done
