set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist_local.py -x -q -m "gpu and not slow" 2>&1 | tail -2
for d in 1 0; do HMG_DEFER_X=$d timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/j_bench_$d.json 2>gpurun_out/j_bench_$d.err; echo "bench $d exit $?"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/j_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu $?"
