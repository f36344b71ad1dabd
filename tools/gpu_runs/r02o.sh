# NEXT-4 buoyancy: parity
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02o_build.log 2>&1; echo "build $?"
timeout 1500 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_parity.py -x -q > gpurun_out/r02o_pytest.log 2>&1; echo "pytest $?"
