set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/ac_bench.json 2>gpurun_out/ac_bench.err; echo "bench exit $?"
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ac_c4.json 2>gpurun_out/ac_c4.err; echo "c4 exit $?"
