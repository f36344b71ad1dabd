set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/f_pytest.log
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench exit $?"
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/f_c4.json 2> gpurun_out/f_c4.err; echo "c4 exit $?"
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/f_c1.json 2> gpurun_out/f_c1.err; echo "c1 exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/f_ncu.log 2>&1; echo "ncu exit $?"
