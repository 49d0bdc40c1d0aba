# A/B of prebuilt variants on selected workloads: VARIANTS="A B" ONLY="northern/pid_pump,..." ABDIR=x bash tools/ab2.sh
mkdir -p gpurun_out/${ABDIR:-ab}
for r in 1 2; do for v in ${VARIANTS}; do
  GLUCOSIM_LIB=build_v$v/libglucosim.so python tools/ab_kernel.py $v ${ONLY} >> gpurun_out/${ABDIR:-ab}/log.jsonl 2>> gpurun_out/${ABDIR:-ab}/err.txt
done; done
