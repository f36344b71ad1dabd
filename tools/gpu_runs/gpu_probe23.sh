set -x
HMG_ST_G4=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu" -k "full_size_c2 or streamed" 2>&1 | tail -2
for g in 1 0; do HMG_ST_G4=$g timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/u_bench_$g.json 2>gpurun_out/u_bench_$g.err; echo "bench $g exit $?"; done
