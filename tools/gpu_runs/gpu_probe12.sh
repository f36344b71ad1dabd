set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "streamed or c4 or C4 or layer" 2>&1 | tail -2
for r in 1 0; do HMG_RES_WARPS=$r timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/l_c4_$r.json 2> gpurun_out/l_c4_$r.err; echo "c4 $r exit $?"; done
