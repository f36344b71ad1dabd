set -x
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/x_c4.json 2> gpurun_out/x_c4.err; echo "c4 exit $?"
for pf in 2 4; do HMG_L2PF=$pf timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/x_bench_pf$pf.json 2>/dev/null; echo "pf $pf exit $?"; done
timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/x_bench.json 2>/dev/null; echo "bench exit $?"
