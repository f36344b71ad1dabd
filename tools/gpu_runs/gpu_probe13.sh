set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist_local.py -x -q -m gpu 2>&1 | tail -3
for e in 1 0; do HMG_EDGE_H=$e timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/m_bench_$e.json 2>gpurun_out/m_bench_$e.err; echo "bench $e exit $?"; done
