set -x
HMG_EDGE_MIN_DOFS=1000000 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist_local.py -x -q -m "gpu and not slow" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" 2>&1 | tail -2
timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/r_bench.json 2>gpurun_out/r_bench.err; echo "bench exit $?"
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r_c4.json 2>gpurun_out/r_c4.err; echo "c4 exit $?"
