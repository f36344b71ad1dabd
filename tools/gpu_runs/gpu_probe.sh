set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_lat tools/micro/fp64_lat.cu && /tmp/fp64_lat
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "apply or layer or c1 or C1" 2>&1 | tail -3
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/p_c1.json 2> gpurun_out/p_c1.err; echo "c1 exit $?"
timeout 600 python tools/micro/st_timing.py 2>&1 | tail -5
