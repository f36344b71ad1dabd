set -x
free -g | head -2
timeout 900 python -m pytest tests/test_gpu_mixed.py -x -q -m "gpu and not slow" 2>&1 | tail -25
timeout 1200 python -m pytest tests/test_gpu_mixed.py -x -q -m "slow" --durations=3 2>&1 | tail -15
