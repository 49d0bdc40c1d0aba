# HEAD check on one B200: GPU tests, smoke, bench line.  Output under gpurun_out/$1/.
O=gpurun_out/${1:-r02d}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest exit $?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_pid.json 2> $O/bench_pid.err
echo done > $O/DONE
