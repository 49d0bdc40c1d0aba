# Round-2 measurement set G (one gpurun call, final round-2 kernel).  Output under gpurun_out/r02g/
set -x
O=gpurun_out/r02g; mkdir -p $O
python bench.py --steps 20 --warmup 3 > $O/bench_pid.json 2> $O/bench_pid.err
python bench.py --controller dual_hormone --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_dual.json 2> $O/bench_dual.err
python bench.py --workload trial1m --steps 2 --warmup 1 > $O/trial1m.json 2> $O/trial1m.err
python bench.py --workload trial1m --patients 125000 --steps 3 --warmup 1 > $O/trial1m_125k.json 2> $O/trial1m_125k.err
python tools/run_configs.py --out $O/configs_pid.json > $O/configs_pid.log 2>&1
python tools/run_configs.py --controller dual_hormone --only C1,C2,C2N --out $O/configs_dual.json > $O/configs_dual.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"^fast_kernel" -c 1 -o $O/fast_pid python tools/prof_fast.py 100000 4 1 three_meal pid_pump > $O/ncu_full_pid.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"^fast_kernel" -c 1 -o $O/fast_dual python tools/prof_fast.py 100000 4 1 three_meal dual_hormone > $O/ncu_full_dual.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sampler_kernel -c 1 -o $O/sampler python tools/prof_fast.py 1000000 1 1 three_meal pid_pump > $O/ncu_sampler.log 2>&1

python tools/time_sampler.py > $O/sampler.jsonl 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err
echo done > $O/DONE
