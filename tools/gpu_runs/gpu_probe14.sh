set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "apply or sweep or vcycle or pcg or full_size or streamed" 2>&1 | tail -2
HMG_EDGE_MIN_DOFS=1000000 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" 2>&1 | tail -2
for e in 1 0; do HMG_EDGE_H=$e timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/n_bench_$e.json 2>gpurun_out/n_bench_$e.err; echo "bench $e exit $?"; done
for e in 1 0; do HMG_EDGE_H=$e timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/n_c4_$e.json 2>gpurun_out/n_c4_$e.err; echo "c4 $e exit $?"; done
