mkdir -p gpurun_out/${ABDIR:-ab1}
for r in 1 2; do for v in ${VARIANTS:-A B C D E}; do
  GLUCOSIM_LIB=build_v$v/libglucosim.so python tools/ab_kernel.py $v >> gpurun_out/${ABDIR:-ab1}/log.jsonl 2>> gpurun_out/${ABDIR:-ab1}/err.txt
done; done
