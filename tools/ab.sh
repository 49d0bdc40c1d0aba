# A/B timing of prebuilt library variants: bash tools/ab.sh A C D ...
mkdir -p gpurun_out/ab
for r in 1 2; do
for v in "$@"; do
  echo "== $v" >> gpurun_out/ab/log.txt
  GLUCOSIM_LIB=build_v$v/libglucosim.so python tools/prof_fast.py 100000 4 5 three_meal pid_pump 2>&1 | tail -2 >> gpurun_out/ab/log.txt
  GLUCOSIM_LIB=build_v$v/libglucosim.so python tools/prof_fast.py 100000 4 4 three_meal dual_hormone 2>&1 | tail -1 >> gpurun_out/ab/log.txt
done; done
