set -x
HMG_EDGE_MIN_DOFS=1000000 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist_local.py -x -q -m "gpu and not slow" 2>&1 | tail -2
for e in 1 0; do HMG_EDGE_RESID=$e timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/p_bench_$e.json 2>gpurun_out/p_bench_$e.err; echo "bench $e exit $?"; done
HMG_EDGE_RESID=1 timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/p_c4.json 2>gpurun_out/p_c4.err; echo "c4 exit $?"
