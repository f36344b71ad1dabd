set -x
HMG_X_BLOCKS=148 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_dist_local.py -x -q -m "gpu and not slow" 2>&1 | tail -2
for b in 96 148 200 296 444; do HMG_X_BLOCKS=$b timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/w_bench_$b.json 2>gpurun_out/w_bench_$b.err; echo "bench $b exit $?"; done
