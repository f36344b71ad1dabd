set -x
HMG_RESID_ST_ALL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" 2>&1 | tail -2
for a in 1 0; do HMG_RESID_ST_ALL=$a timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/z_bench_$a.json 2>gpurun_out/z_bench_$a.err; echo "bench $a exit $?"; done
HMG_RESID_ST_ALL=1 timeout 600 python tools/level_breakdown.py C2b 2>&1 | tail -14
