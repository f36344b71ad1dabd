set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "coop or coarse or vcycle or pcg" 2>&1 | tail -3
timeout 600 python tools/micro/coop_timing.py 4 2>&1 | tail -4
for r in 4 3 5; do HMG_COOP_REF=$r timeout 300 python tools/vc_time.py C2b; done
timeout 300 python tools/vc_time.py C2b
