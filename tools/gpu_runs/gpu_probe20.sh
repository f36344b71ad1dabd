set -x
HMG_EDGE_MIN_DOFS=1000000 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist_local.py tests/test_gpu_mixed.py -x -q -m "gpu and not slow" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" 2>&1 | tail -2
timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/s_bench.json 2>gpurun_out/s_bench.err; echo "bench exit $?"
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/s_c1.json 2>gpurun_out/s_c1.err; echo "c1 exit $?"
