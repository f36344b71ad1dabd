set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/g_pytest.log
timeout 900 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo "bench exit $?"
tail -3 gpurun_out/g_bench.err
