set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/l_pytest.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/l_pytest.log
timeout 900 python bench.py > gpurun_out/l_bench.json 2> gpurun_out/l_bench.err; echo "bench exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke $?"
