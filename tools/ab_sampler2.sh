# Sampler variants (built here by tools/build_sampler_variant.sh): timing of each, log in gpurun_out/abs2/
mkdir -p gpurun_out/abs2
for v in ${VARIANTS}; do
  echo "== $v" >> gpurun_out/abs2/log.txt
  GLUCOSIM_LIB=build_v$v/libglucosim.so timeout 300 python tools/time_sampler.py >> gpurun_out/abs2/log.txt 2>&1
done
