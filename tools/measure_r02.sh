# Round-2 measurement set (one gpurun call).  Output under gpurun_out/r02/.
set -x
O=gpurun_out/r02; mkdir -p $O
nproc > $O/nproc.txt
timeout 900 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize.py > $O/sanitize_memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize.py > $O/sanitize_racecheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize.py > $O/sanitize_synccheck.log 2>&1
python bench.py > $O/bench_pid.json 2> $O/bench_pid.err
python bench.py --controller dual_hormone > $O/bench_dual.json 2> $O/bench_dual.err
timeout 1200 python tools/time_reference_cpu.py ${REF_N:-20000} 4 > $O/reference_cpu.json 2> $O/reference_cpu.err
python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1
echo done > $O/DONE
