set -x
HMG_X_BLOCKS=32 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" -k "pcg or host" 2>&1 | tail -2
for b in 0 16 32 64 148; do HMG_X_BLOCKS=$b timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/v_bench_$b.json 2>gpurun_out/v_bench_$b.err; echo "bench $b exit $?"; done
