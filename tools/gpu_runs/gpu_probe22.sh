set -x
for m in 16777216 4000000 1000000; do HMG_EDGE_MIN_DOFS=$m timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/t_bench_$m.json 2>gpurun_out/t_bench_$m.err; echo "bench $m exit $?"; done
