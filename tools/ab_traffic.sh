# DRAM bytes of one fused-kernel launch (100k x 4 w, PID) per library variant: bash tools/ab_traffic.sh A J ...
mkdir -p gpurun_out/ab
for v in "$@"; do
  echo "== $v" >> gpurun_out/ab/traffic.txt
  GLUCOSIM_LIB=build_v$v/libglucosim.so ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:fast_kernel -c 1 python tools/prof_fast.py 100000 4 1 three_meal pid_pump 2>&1 \
    | grep -E 'dram__|gpu__time' >> gpurun_out/ab/traffic.txt
done
