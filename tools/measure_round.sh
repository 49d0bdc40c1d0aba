# Round measurement set (one gpurun call): bench lines, configs, launch list, ncu captures.
mkdir -p gpurun_out/m
python bench.py > gpurun_out/m/bench_pid.json 2> gpurun_out/m/bench_pid.err
python bench.py --controller dual_hormone > gpurun_out/m/bench_dual.json 2> gpurun_out/m/bench_dual.err
python bench.py --workload trial1m > gpurun_out/m/trial1m.json 2> gpurun_out/m/trial1m.err
python bench.py --workload trial1m --patients 125000 > gpurun_out/m/trial1m_125k.json 2> gpurun_out/m/trial1m_125k.err
python tools/run_configs.py --out gpurun_out/m/configs_pid.json > gpurun_out/m/configs_pid.log 2>&1
python tools/run_configs.py --controller dual_hormone --out gpurun_out/m/configs_dual.json > gpurun_out/m/configs_dual.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/m/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fast_kernel -c 1 -o gpurun_out/m/fast_pid python tools/prof_fast.py 100000 4 1 three_meal pid_pump > gpurun_out/m/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fast_kernel -c 1 -o gpurun_out/m/fast_dual python tools/prof_fast.py 100000 4 1 three_meal dual_hormone > gpurun_out/m/ncu_full_dual.log 2>&1
echo done > gpurun_out/m/DONE
