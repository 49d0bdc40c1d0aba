mkdir -p gpurun_out/abs
for v in ${VARIANTS}; do
  echo "== $v" >> gpurun_out/abs/log.txt
  GLUCOSIM_LIB=build_v$v/libglucosim.so python tools/time_sampler.py >> gpurun_out/abs/log.txt 2>&1
done
