set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist_local.py -x -q -m "gpu and not slow" 2>&1 | tail -2
timeout 800 python tools/micro/coop_timing.py 4 2>&1 | tail -3
timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/aa_bench.json 2>gpurun_out/aa_bench.err; echo "bench exit $?"
timeout 600 python tools/level_breakdown.py C2b 2>&1 | tail -14
