set -x
HMG_APPLY_CTAS=3 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" -k "apply or pcg or vcycle or edge" 2>&1 | tail -2
for c in 3 2; do HMG_APPLY_CTAS=$c timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/ab_bench_$c.json 2>gpurun_out/ab_bench_$c.err; echo "bench $c exit $?"; done
for c in 3 2; do HMG_APPLY_CTAS=$c timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/ab_c1_$c.json 2>/dev/null; echo "c1 $c exit $?"; done
